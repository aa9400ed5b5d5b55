"""In-kernel cycle accounting of the band kernel (ri_tc.cu, RC_TC_PROF counters).

Builds a profiling variant of the library (ri_tc.cu with -DRC_TC_PROF=1, the other objects
from the normal build) into tools/variants/, runs one layer config a few times and prints,
per CTA on average: each MMA warp's total / waiting-for-D / waiting-for-X / waiting-for-W /
issuing cycles, the epilogue warp's total / waiting-for-D / finalize cycles and the
producers' waits.  Experiment tooling; the shipped library has the counters compiled out.

    python tools/tc_kernel_profile.py build [VARIANT -DNAME=V ...]   # here (nvcc cross-compiles)
    python tools/tc_kernel_profile.py run [--lib VARIANT] N CIN H W COUT GROUP R POOL G [precision]
"""
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VAR = os.path.join(ROOT, "tools", "variants")
NAMES = ["mma0 total", "mma0 wait D", "mma0 wait X", "mma0 wait W", "mma0 issue",
         "mma1 total", "mma1 wait D", "mma1 wait X", "mma1 wait W", "mma1 issue",
         "epi total", "epi wait Dfull", "epi finalize", "prod0 wait Wslot", "prod0 wait Xslot",
         "prod1 wait Wslot", "epi8 total", "epi8 wait Dfull", "epi8 finalize"]


def lib_path(variant="prof"):
    return os.path.join(VAR, f"librotconv_{variant}.so")


def build(variant="prof", defines=()):
    from paper_2512_08888_b200 import build as B
    B.build()
    os.makedirs(VAR, exist_ok=True)
    obj = os.path.join(VAR, f"ri_tc_{variant}.o")
    prof = [] if "-DRC_TC_PROF=0" in defines else ["-DRC_TC_PROF=1"]  # =0: a timing-only variant
    subprocess.check_call([B.NVCC, *B.ARCH, *[f for f in B.FLAGS if f not in ("-Xptxas", "-v")],
                           *prof, *defines, "-c", os.path.join(B.CSRC, "ri_tc.cu"), "-o", obj])
    objs = [os.path.join(B.BUILD, f) for f in sorted(os.listdir(B.BUILD))
            if f.endswith(".o") and f != "ri_tc.o"] + [obj]
    subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-o", lib_path(variant), *objs, "-lcublas"])
    print(lib_path(variant))


def run(a):
    import torch
    from paper_2512_08888_b200 import _lib
    variant = "prof"
    if a[0] == "--lib":
        variant, a = a[1], a[2:]
    _lib.LIB_PATH = lib_path(variant)
    try:
        C.CDLL(_lib.LIB_PATH).rc_tc_prof
        prof = True
        _lib.SIGNATURES["rc_tc_prof"] = (C.c_int, [C.c_void_p, C.c_int, C.c_int])
    except AttributeError:  # a timing-only variant (-DRC_TC_PROF=0)
        prof = False
    import paper_2512_08888_b200 as P
    n, cin, h, w, cout = map(int, a[:5])
    group, R, pool, g = a[5], int(a[6]), a[7], int(a[8])
    prec = a[9] if len(a) > 9 else "auto"
    desc = P.Desc(n, cin, h, w, cout, 3, group, R, pool, g, "scatter", prec)
    x = torch.rand((n, cin, h, w), device="cuda") * 2 - 1
    w0 = (torch.rand((cout, cin, 3, 3), device="cuda") * 2 - 1) * 0.05
    w1 = (torch.rand((cout, cin, 3, 3), device="cuda") * 2 - 1) * 0.05 if group == "steer" else None
    bank = P.bank_precompute(desc, w0, w1)
    L = _lib.lib()
    reps = 5 if prof else 20
    for _ in range(3):
        P.ri_conv_forward(desc, x, bank)
    torch.cuda.synchronize()
    if prof:
        L.rc_tc_prof(None, 0, 1)
    times = []
    for _ in range(1 if prof else 5):
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(reps):
            P.ri_conv_forward(desc, x, bank)
        a1.record()
        torch.cuda.synchronize()
        times.append(a0.elapsed_time(a1) / reps)
    ms = sorted(times)[len(times) // 2]
    if not prof:
        print(f"[{variant}] {desc.kernel_name()} {ms:.4f} ms per launch (incl. x_pack; median of {len(times)} x {reps})")
        return
    buf = (C.c_ulonglong * (1024 * 32))()
    L.rc_tc_prof(buf, 1024 * 32, 0)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    ctas = min(sms, (cout + 127) // 128 * n)
    tot = [sum(buf[c * 32 + i] for c in range(ctas)) / ctas / reps for i in range(len(NAMES))]
    print(f"[{variant}] {desc.kernel_name()} {ms:.3f} ms per launch (incl. x_pack), {ctas} CTAs; per CTA per launch, "
          f"Mcycles (share of the MMA warp 0 total):")
    for i, nm in enumerate(NAMES):
        print(f"  {nm:18s} {tot[i] / 1e6:8.3f}  {tot[i] / max(tot[0], 1):6.3f}")


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2] if len(sys.argv) > 2 else "prof", sys.argv[3:])
    else:
        run(sys.argv[2:])
