"""Benchmark of the fused RI scatter-conv layer (the north-star hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3|c4|c1] [--impl ours|reference]

One step = one layer forward over one batch (BASELINE.json metric: "RI-conv layer ms &
effective TFLOP/s").  Default workload C3: 16x16 input, Cin 256 -> Cout 1024, steerable
R=8 (B=2 bases), subgroup-4 max pooling + argmax + bias, batch 256 per GPU (weak
scaling: every rank runs its own 256-image shard; no data-path collective).

Rank 0 prints ONE JSON line.  value = whole-job effective TFLOP/s (cuDNN-equivalent
2*N*H*W*K^2*Cin*Cout*R over all ranks / max-over-ranks device time); ms_per_step = layer
ms; roofline = algorithmic FLOPs of the fused kernel per launch / its CUDA-event time
vs the measured bf16 tensor peak; e2e = the same metric through the C-ABI host entry
point (rc_ri_conv_forward_host) with pinned host buffers, H2D + D2H inside the timed
region; cpu_baseline = the CPU path on a bounded sample, timed on this host.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

STRONG = {"c4", "c5"}  # fixed global batch split over the ranks; c1/c3: fixed batch per rank
WORKLOADS = {
    # name: (n per rank, cin, h, w, cout, k, group, R, pool, pool_group, label)
    "c3": (256, 256, 16, 16, 1024, 3, "steer", 8, "subgroup", 4,
           "C3: RI conv 16x16x256->1024, steerable R=8 (2 bases), subgroup-4 max+argmax+bias"),
    # C4: global batch 512 sharded over the ranks (BASELINE.json: "batch 512, batch-sharded
    # over 2/4/8 GPUs") -> strong scaling
    "c4": (512, 128, 32, 32, 512, 3, "steer", 16, "subgroup", 4,
           "C4: RI conv 32x32x128->512, steerable R=16 (4 bases), subgroup-4 max+argmax+bias, "
           "global batch 512 sharded over the GPUs"),
    "c1": (32, 64, 8, 8, 256, 3, "single", 1, "none", 1,
           "C1: single-orientation scatter conv 8x8x64->256"),
    # C5: the multi-layer RI classifier (paper_2512_08888_b200/stack.py), global batch 1024
    # split over the ranks (strong scaling)
    "c5": (1024, 3, 64, 64, 10, 3, "stack", 8, "subgroup", 4,
           "C5: RI classifier stack 64x64x3, 3 blocks (RI steer R=8 subgroup-4 + conv + ReLU + "
           "maxpool), widths 64/128/256, GAP + linear head"),
    # C2: the paper's Appendix-A grid, one step = every cell once (its largest cell is the
    # tuple's shape, used for the CPU sample and the roofline)
    "c2": (32, 256, 16, 16, 1024, 3, "single", 1, "none", 1,
           "C2: single-orientation scatter conv grid, inputs 4x4/8x8/16x16 x Cin 4..256 x Cout "
           "256/512/1024, batch 32 per cell (63 cells per step)"),
}
C2_SIZES, C2_CINS, C2_COUTS = (4, 8, 16), (4, 8, 16, 32, 64, 128, 256), (256, 512, 1024)



# Compute peaks MEASURED_PEAKS.json does not hold, measured on a B200 of this pool by
# tools/peak_probe.cu (profiles/r02/peaks/peak_probe.jsonl): FP32 FMA on the CUDA cores (FFMA
# and packed FFMA2 reach the same rate), tcgen05 kind::tf32 and kind::f16 issue-rate peaks
# of an operand-resident MMA loop (M = 128, N = 256) at 1965 MHz.
PEAKS_SRC = "tools/peak_probe.cu, profiles/r02/peaks/peak_probe.jsonl"
FFMA_PEAK = 72.7
PROBED_PEAKS = {"ffma_tflops": 71.75, "ffma2_tflops": 72.72, "tcgen05_tf32_tflops": 1115.0,
                "tcgen05_bf16_loop_tflops": 2229.0, "source": PEAKS_SRC}

def arith_dtype(kernel: str) -> str:
    """Arithmetic the timed kernel computes in (not a precision claim)."""
    if kernel.startswith("tc_") and kernel.endswith("bf16x3"):
        return "bf16x3 (3 bf16 MMA products, f32 accumulate)"
    if kernel.startswith("tc_"):
        return "bf16 (f32 accumulate)"
    return "f32"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("bf16_tflops", 1590.0), d.get("hbm_gbs", 6650.0), "measured"
    return 1590.0, 6650.0, "fallback"


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: NVML polled every 2 ms
    from a thread, plus explicit sample() calls while queued GPU work is still running (a
    sub-millisecond timed region still gets samples).  Falls back to nvidia-smi -lms 10."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.nvml = None
        self.rows: list = []
        self.lines: list[str] = []
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[self.index]) if vis and vis.split(",")[0].isdigit() else self.index
            self.h = N.nvmlDeviceGetHandleByIndex(phys)
            self.nvml = N
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "10"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def sample(self):
        if self.nvml is None:
            return
        N = self.nvml
        try:
            sm = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
            mx = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            bits = [0x8, 0x40, 0x20, 0x4]  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
            self.rows.append((float(sm), float(mx), ["Active" if r & b else "Not Active" for b in bits]))
        except Exception:
            pass

    def _poll(self):
        while not self.stop.is_set():
            self.sample()
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = list(self.rows)
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) >= 9:
                try:
                    rows.append((float(f[1]), float(f[2]), f[5:9]))
                except ValueError:
                    pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({self.NAMES[i] for _, _, fl in rows for i, v in enumerate(fl) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows),
                "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def cpu_reference(wl, threads: int, target_s: float = 12.0, kind: str = "reference", m0: int | None = None):
    """The CPU path on a bounded image sample, timed on this host with every core.

    kind "reference": the reference's own code -- the unmodified tiled_scatter_conv
    (scatter_conv.hpp:330-368, compiled from /root/reference by oracle/Makefile into
    oracle/_ref) once per orientation slice (R x tiled_scatter_conv: the reference has no
    reuse path), plus the SPEC pooling and bias (oracle/ref_shim.cpp ref_ri_batch_f).
    kind "port": the oracle's C restatement of the paper's reuse loop (one dot per tap,
    scattered to the 4 rotations; bit-identical to the reference slices,
    tests/test_oracle_ref.py).  The sample starts at m0 (default: one image per thread) and
    doubles until it takes >= target_s / 4.  Returns (eff TFLOP/s, dict)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    n, cin, h, w, cout, k, g, R, pool, pg, _ = wl
    rng = np.random.default_rng(0)
    s = 1 / np.sqrt(cin * k * k)
    if kind == "reference" and not O.ref_available():
        kind = "port"
    fx = rng.uniform(-s, s, (cout, cin, k, k)).astype(np.float32)
    fy = rng.uniform(-s, s, (cout, cin, k, k)).astype(np.float32)
    bias = rng.uniform(-0.1, 0.1, cout).astype(np.float32)

    def run(m):
        x = rng.uniform(-1, 1, (m, cin, h, w)).astype(np.float32)
        d = O.Desc(m, cin, h, w, cout, k, g, R, pool, pg)
        t0 = time.perf_counter()
        if kind == "reference":
            O.ref_ri_batch(d, x, fx, fy, bias, nthreads=threads)
        else:
            O.ri_forward(d, x, fx, fy, bias, nthreads=threads)
        return time.perf_counter() - t0

    m = m0 or threads
    dt = run(m)
    while dt < target_s / 4 and m < n:
        m = min(n, m * 2)
        dt = run(m)
    eff = 2.0 * m * h * w * k * k * cin * cout * R
    what = ("R x unmodified tiled_scatter_conv per image + SPEC pooling/bias (oracle/_ref)" if kind == "reference"
            else "oracle C port of the reuse loop (oracle/librc_oracle.so)")
    return eff / dt / 1e12, {"cores": threads, "kind": kind, "images": m, "sample_s": dt,
                             "sample": f"{m} of {n} images x all {cout} output channels in {dt:.2f} s on "
                                       f"{threads} threads: {what}",
                             "ms_full_layer_extrapolated": dt * n / m * 1e3}


def workload_config(args, wl, world: int) -> dict:
    """The workload a line is quoted on -- identical in both arms (ours and --impl reference)."""
    n, cin, h, w, cout, k, g, R, pool, pg, label = wl
    strong = args.workload in STRONG
    return {"workload": label, "global_batch": n if strong else n * world,
            "n_per_gpu": -(-n // world) if strong else n, "c_in": cin, "h": h, "w": w, "c_out": cout, "k": k,
            "group": g, "orientations": R, "pool": pool, "pool_group": pg,
            "parallelism": f"batch-sharded dp{world}"}


def run_reference(args, wl):
    """--impl reference: the reference's own CPU implementation of the path on this host's
    cores (rank 0 only), every step a bounded sample of the workload (one image per host
    thread, R x tiled_scatter_conv each), same metric / unit / config as our arm."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", args.gpus))
    threads = os.cpu_count() or 1
    vals, secs, info = [], [], None
    for i in range(args.warmup + args.steps):
        v, info = cpu_reference(wl, threads, target_s=0.0, kind="reference")
        if i >= args.warmup:
            vals.append(v)
            secs.append(info["sample_s"])
    v = statistics.median(vals)
    ms = statistics.median(secs) * 1e3
    out = {"impl": "reference", "metric": "RI-conv layer effective TFLOP/s", "value": v,
           "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": ms, "ms_per_step_is": f"measured wall time of one step = a {info['images']}-image sample",
           "ms_full_layer_extrapolated": info["ms_full_layer_extrapolated"] * (world if args.workload not in STRONG else 1),
           "higher_is_better": True,
           "scaling": "strong" if args.workload in STRONG else "weak", "vs_baseline": None,
           "dtype": "f32", "data": "synthetic (uniform[-1,1) inputs, uniform/sqrt(Cin*K^2) weights, random init)",
           "config": workload_config(args, wl, world),
           "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": threads, "kind": info["kind"],
                            "sample": info["sample"]},
           "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "note": "the reference has no GPU path: one host runs it; value = effective FLOPs of the sample / its "
                   "wall time (rate is linear in images)"}
    print(json.dumps(out), flush=True)


def smem_traffic(desc, kernel: str):
    """Shared-memory bytes one launch of the band kernel (ri_tc.cu) moves, from its geometry;
    None for other kernels.  Per K-step (16 ci of one chunk):
      * 16-wide carry bands (tc_k3w16; N = 64 px, no halo): bf16x3 reads A = Wh once (the
        N = 128 Wh x [Xh | Xl] MMA) + Wl once (Wl x Xh) and B = 128 + 64 rows x 32 B; bf16
        reads A once and B = 64 rows; the TMA writes parts x 4 KB of weights.  The X band
        (parts x NC x 64 px x 128 B) is written once per (base, band) unit.
      * strips of wider images (tc_k3strip): the same carry bands over 16-column strips, 4
        input rows x 18 columns (halo columns only), N = 72; bf16x3 as three N = 72 MMAs (Ah
        twice + Al once, Xh twice + Xl once); X written once per (base, band) unit."""
    if not (kernel.startswith("tc_k3w16") or kernel.startswith("tc_k3strip")):
        return None
    three = kernel.endswith("bf16x3")
    parts = 2 if three else 1
    n, h, w, cin, cout = desc.n, desc.h, desc.w, desc.c_in, desc.c_out
    NB = {"single": 1, "p4": 1, "p4m": 2, "steer": desc.orientations // 4}[desc.group]
    NC = (cin + 63) // 64
    NCT = (cout + 127) // 128
    if kernel.startswith("tc_k3w16"):
        nbk = (h + 3) // 4
        kstep = (2 * 4096 + (128 + 64) * 32 + 2 * 4096) if three else (4096 + 64 * 32 + 4096)
        per_item = NB * nbk * (9 * NC * 4 * kstep + parts * NC * 64 * 128)
    else:
        pa = 3 if three else 1
        bands = ((h + 3) // 4) * (w // 16)
        kstep = pa * 4096 + pa * 72 * 32 + parts * 4096
        per_item = NB * bands * (9 * NC * 4 * kstep + parts * NC * 72 * 128)
    return per_item * n * NCT


def smem_roofline(desc, kernel_ms):
    """The band kernel's binding roofline: shared-memory bandwidth (SS operand reads + TMA
    writes), 128 B/cycle/SM x 148 SMs at the max SM clock (37.2 TB/s)."""
    b = smem_traffic(desc, desc.kernel_name())
    if b is None or not kernel_ms:
        return None
    ach = b / (kernel_ms * 1e-3) / 1e12
    peak = 128 * 148 * 1.965e9 / 1e12
    return {"bytes_per_launch": b, "achieved": ach, "peak": peak, "unit": "TB/s", "frac": ach / peak,
            "note": "SS MMA operand reads + TMA weight/X writes per launch (bench.smem_traffic), / main-kernel time"}


def backward_context(P, desc, x, bank, y, am, reps=3):
    """The layer's backward (SPEC backward module: pool/ReLU/bias backward, input gradient,
    weight gradient) on the same inputs, CUDA-event timed after one warm-up; context for the
    forward line, not part of the timed step."""
    import torch
    gy = torch.rand(y.shape, device=x.device)
    run = lambda: P.ri_conv_backward(desc, x, bank, gy, y, am)
    run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        run()
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / reps
    return {"ms": ms,
            "grads": "dx, dW (f_x, f_y for steer), dbias",
            "path": "rc_ri_conv_backward: pool backward, implicit-GEMM input gradient, tcgen05 weight gradient"
            if desc.kernel_name().startswith("tc_") else "rc_ri_conv_backward (fp32: CUDA-core input pass, SGEMM weights)"}


def cudnn_context(P, desc, x, fx, fy, ours_ms, args):
    """Context only (not the product path): the same R orientation slices
    as R separate cuDNN convolutions on the rotated kernels (the paper's cuDNN RI pipeline),
    unpooled, FP32 and TF32-allowed, on this B200.  Our step above also pools + biases."""
    import torch
    import torch.nn.functional as F
    k, R = desc.k, desc.orientations
    kern = P.rotconv.build_orientation_bank_from(desc, fx, fy if desc.group == "steer" else None)
    wcat = torch.flip(kern, dims=(3, 4)).reshape(R * desc.c_out, desc.c_in, k, k).contiguous()
    torch.backends.cudnn.benchmark = True
    out = {}
    for name, tf32 in (("fp32", False), ("tf32", True)):
        torch.backends.cudnn.allow_tf32 = tf32
        for _ in range(3):
            F.conv2d(x, wcat, padding=k // 2)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            F.conv2d(x, wcat, padding=k // 2)
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        out[f"cudnn_{name}_ms"] = statistics.median(ts)
    torch.backends.cudnn.allow_tf32 = False
    out["ours_ms"] = ours_ms
    out["speedup_vs_cudnn_fp32"] = out["cudnn_fp32_ms"] / ours_ms
    out["speedup_vs_cudnn_tf32"] = out["cudnn_tf32_ms"] / ours_ms
    out["note"] = ("R separate cuDNN convs (unpooled, batch in HBM) vs this repo's fused layer "
                   "(reuse scatter + subgroup pooling + argmax + bias); context, not the product path")
    return out


def _stack_cpu_sample(threads, n_img=2):
    """Oracle composition of the C5 stack on a bounded sample (tests/test_gpu_stack.py)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle as O
    import torch
    from paper_2512_08888_b200.stack import RIStack, StackSpec
    from test_gpu_stack import oracle_stack
    stack = RIStack(StackSpec(), "cpu" if not torch.cuda.is_available() else "cuda", seed=5)
    x = np.random.default_rng(0).uniform(-1, 1, (n_img, 3, 64, 64)).astype(np.float32)
    t0 = time.perf_counter()
    oracle_stack(O, stack, x, nthreads=threads)
    dt = time.perf_counter() - t0
    return stack, dt, n_img


def stack_config(args, wl, world: int) -> dict:
    """C5 workload config -- identical in both arms."""
    return {"workload": wl[-1], "global_batch": wl[0], "batch_per_gpu": -(-wl[0] // world),
            "image": "3x64x64", "widths": [64, 128, 256], "orientations": 8, "pool": "subgroup", "pool_group": 4,
            "parallelism": f"batch-sharded dp{world}"}


def run_stack_reference(args, wl):
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    vals = []
    for i in range(args.warmup + args.steps):
        stack, dt, m = _stack_cpu_sample(threads)
        if i >= args.warmup:
            vals.append(stack.eff_flops(m) / dt / 1e12)
    v = statistics.median(vals)
    n = wl[0]
    out = {"impl": "reference", "metric": "RI classifier forward effective TFLOP/s", "value": v,
           "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": stack.eff_flops(n) / (v * 1e12) * 1e3, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": stack_config(args, wl, int(os.environ.get("WORLD_SIZE", args.gpus))),
           "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": threads, "kind": "port",
                            "sample": "2 images through the whole stack, linear in images"},
           "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def run_stack(args, wl):
    """C5: the whole classifier forward per step; global batch split over the ranks."""
    import torch
    import torch.distributed as dist
    import paper_2512_08888_b200 as P  # noqa: F401
    from paper_2512_08888_b200.stack import RIStack, StackSpec

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        dist.init_process_group("nccl", device_id=dev)
    n_total = wl[0]
    b, e = P.shard_range(n_total, world, rank)
    n = e - b
    stack = RIStack(StackSpec(precision=args.precision), dev, seed=5)  # same weights on every rank
    gen = torch.Generator(device=dev).manual_seed(99 + rank)
    x = (torch.rand((n, 3, 64, 64), generator=gen, device=dev) * 2 - 1).contiguous()
    flush = torch.empty(512 * 1024 * 1024 // 4, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        stack.graph_forward(x)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))
            ev[i][0].record(stream)
            stack.graph_forward(x)
            ev[i][1].record(stream)
        clk.sample()  # the queued steps are still running on the GPU
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    times = [a.elapsed_time(bb) for a, bb in ev]
    tot = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
    per_rank = [tot.clone() for _ in range(world)]
    if world > 1:
        dist.all_gather(per_rank, tot)
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    per_rank_ms = [round(t.item() / args.steps, 4) for t in per_rank]
    ms = tot.item() / args.steps
    eff_total = stack.eff_flops(n_total)
    value = eff_total / (ms * 1e-3) / 1e12
    # per-layer device time (untimed pass) -> the dominant kernel for the roofline line
    layer_ms = []
    for layer in stack.layers:
        d = layer.desc(n, stack.spec)
        y = torch.empty((n, layer.cout, d.out_orientations, layer.size, layer.size), device=dev)
        am = torch.empty(y.shape, dtype=torch.uint8, device=dev) if d.has_argmax else None
        xin = torch.rand((n, layer.cin, layer.size, layer.size), device=dev)
        bank = stack._bank(layer, d)
        P.ri_conv_forward(d, xin, bank, layer.bias, out=y, argmax=am)
        a, bb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(3):
            P.ri_conv_forward(d, xin, bank, layer.bias, out=y, argmax=am)
        bb.record(stream)
        bb.synchronize()
        layer_ms.append((a.elapsed_time(bb) / 3, d))
    top_ms, top = max(layer_ms, key=lambda t: t[0])
    achieved = top.alg_flops() / (top_ms * 1e-3) / 1e12
    tpeak, _, src = peaks()
    # e2e through the public API: pinned host input -> device, forward, logits -> host
    hx = torch.empty((n, 3, 64, 64), pin_memory=True)
    hx.copy_(x)
    xd = torch.empty_like(x)
    hl = torch.empty((n, stack.spec.classes), pin_memory=True)
    e2e_t = []
    for i in range(max(1, args.e2e_steps) + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        xd.copy_(hx, non_blocking=True)
        hl.copy_(stack.graph_forward(xd), non_blocking=True)
        torch.cuda.synchronize()
        if i:
            e2e_t.append(time.perf_counter() - t0)
    e2e_s = torch.tensor([statistics.mean(e2e_t)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        st, dt, m = _stack_cpu_sample(threads)
        cpu = {"value": st.eff_flops(m) / dt / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": "port",
               "sample": f"{m} images through the whole stack ({dt:.2f} s), linear in images",
               "ms_full_batch_extrapolated": dt * n_total / m * 1e3}
    if rank == 0:
        out = {
            "metric": "RI classifier forward effective TFLOP/s", "value": value, "unit": "TFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "mixed: " + ", ".join(sorted({arith_dtype(k) for k in stack.kernels(n)})),
            "data": "synthetic (uniform[-1,1) images, random-init weights)",
            "config": stack_config(args, wl, world),
            "precision": args.precision, "kernels": stack.kernels(n), "cuda_graph": True,
            "l2": "flushed between timed iterations (512 MB write)",
            "alg_tflops": stack.alg_flops(n_total) / (ms * 1e-3) / 1e12, "per_rank_ms": per_rank_ms,
            "layer_ms": [round(t, 4) for t, _ in layer_ms],
            "roofline": {"bound": "tensor" if top.kernel_name().startswith("tc_") else "fp32-simt",
                         "kernel": top.kernel_name(), "achieved": achieved,
                         "peak": tpeak if top.kernel_name().startswith("tc_") else FFMA_PEAK,
                         "unit": "TFLOP/s",
                         "frac": achieved / (tpeak if top.kernel_name().startswith("tc_") else FFMA_PEAK),
                         "traffic": None,
                         "peak_source": f"{src} bf16 dense (tc) / measured FP32 FFMA peak (simt, {PEAKS_SRC})",
                         "note": "dominant layer of the stack, alg FLOPs / its CUDA-event time"},
            "clocks": clk.summary(),
            "e2e": {"value": eff_total / e2e_s.item() / 1e12, "unit": "TFLOP/s",
                    "h2d_bytes_per_step": int(hx.numel() * 4), "d2h_bytes_per_step": int(hl.numel() * 4),
                    "ms_per_step": e2e_s.item() * 1e3, "path": "RIStack.graph_forward (pinned host in/out)"},
            "gpu_launches": args.steps * stack.launches_per_forward(n),
            "cpu_baseline": cpu,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_grid(args, wl):
    """C2: the Appendix-A grid (63 single-orientation layers, batch 32 each) as one step.

    value = the grid's effective FLOPs / the step's device time, the step being every cell
    once (inputs resident, outputs preallocated, L2 flushed between steps); per cell, the
    device time of one launch (CUDA-graph replays) next to cuDNN FP32 (FMA-only) and TF32 on
    the same tensors (context: the paper's appendix comparison).  Each rank runs the whole
    grid on its own images (weak scaling)."""
    import torch
    import torch.distributed as dist
    import torch.nn.functional as F
    import paper_2512_08888_b200 as P
    from paper_2512_08888_b200 import _lib

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        dist.init_process_group("nccl", device_id=dev)
    n = wl[0]
    gen = torch.Generator(device=dev).manual_seed(4321 + rank)
    cells = []
    for sz in C2_SIZES:
        for cin in C2_CINS:
            for cout in C2_COUTS:
                d = P.Desc(n, cin, sz, sz, cout, 3, "single", 1, "none", 1, "scatter", args.precision)
                x = (torch.rand((n, cin, sz, sz), generator=gen, device=dev) * 2 - 1).contiguous()
                w0 = ((torch.rand((cout, cin, 3, 3), generator=gen, device=dev) * 2 - 1) / np.sqrt(cin * 9)).contiguous()
                cells.append({"desc": d, "x": x, "w": w0, "bank": P.bank_precompute(d, w0),
                              "y": torch.empty((n, cout, 1, sz, sz), device=dev), "size": sz, "cin": cin, "cout": cout})

    def step():
        for c in cells:
            P.ri_conv_forward(c["desc"], c["x"], c["bank"], out=c["y"])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    s0 = torch.cuda.Stream(dev)
    s0.wait_stream(torch.cuda.current_stream(dev))
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s0):
        step()
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=s0):
            step()
    torch.cuda.synchronize()
    flush = torch.empty(512 * 1024 * 1024 // 4, device=dev)
    stream = torch.cuda.current_stream(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))
            ev[i][0].record(stream)
            graph.replay()
            ev[i][1].record(stream)
        clk.sample()
        torch.cuda.synchronize()
    times = [a.elapsed_time(b) for a, b in ev]
    tot = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
    per_rank = [tot.clone() for _ in range(world)]
    if world > 1:
        dist.all_gather(per_rank, tot)
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms = tot.item() / args.steps
    eff = sum(2.0 * n * c["size"] ** 2 * 9 * c["cin"] * c["cout"] for c in cells)
    value = eff * world / (ms * 1e-3) / 1e12

    def graph_ms(fn, reps=20):  # one call's device time: 5 calls per graph replay
        s1 = torch.cuda.Stream(dev)
        s1.wait_stream(torch.cuda.current_stream(dev))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s1):
            fn()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s1):
                for _ in range(5):
                    fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) / 5)
        return statistics.median(ts)

    rows, wins = [], 0
    if rank == 0 and not args.no_cudnn:
        torch.backends.cudnn.benchmark = True
        for c in cells:
            d, x, w0, bank, y = c["desc"], c["x"], c["w"], c["bank"], c["y"]
            wf = torch.flip(w0, dims=(2, 3)).contiguous()  # scatter_conv_multi == conv2d(X, flip W)
            ours = graph_ms(lambda: P.ri_conv_forward(d, x, bank, out=y))
            torch.backends.cudnn.allow_tf32 = False
            ref = F.conv2d(x, wf, padding=1)
            err = ((y[:, :, 0] - ref).abs().max() / ref.abs().max()).item()
            fp32 = graph_ms(lambda: F.conv2d(x, wf, padding=1))
            torch.backends.cudnn.allow_tf32 = True
            tf32 = graph_ms(lambda: F.conv2d(x, wf, padding=1))
            torch.backends.cudnn.allow_tf32 = False
            wins += ours <= fp32
            rows.append([c["size"], c["cin"], c["cout"], d.kernel_name(), round(ours, 5), round(fp32, 5),
                         round(tf32, 5), round(fp32 / ours, 3), float(f"{err:.2e}")])
    big = cells[-1]  # 16x16x256 -> 1024
    L = _lib.lib()
    L.rc_profile_enable(1)
    for _ in range(5):
        P.ri_conv_forward(big["desc"], big["x"], big["bank"], out=big["y"])
    torch.cuda.synchronize()
    L.rc_profile_enable(0)
    kms = (C.c_float * 5)()
    nk = L.rc_profile_collect(kms, 5)
    kernel_ms = statistics.median(kms[:nk]) if nk > 0 else None
    tpeak, hbm, src = peaks()
    tc = big["desc"].kernel_name().startswith("tc_")
    achieved = big["desc"].alg_flops() / (kernel_ms * 1e-3) / 1e12 if kernel_ms else None
    # e2e: every cell through the C-ABI host entry (pinned buffers, H2D + D2H per cell)
    hbuf = []
    for c in cells:
        d = c["desc"]
        hbuf.append((d.c(), c["x"].cpu().pin_memory(), c["w"].cpu().pin_memory(),
                     torch.empty(tuple(c["y"].shape), pin_memory=True)))
    pp = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None

    def e2e_step():
        for cd, hx, hw, hy in hbuf:
            _lib.check(L.rc_ri_conv_forward_host(C.byref(cd), pp(hx), pp(hw), None, None, pp(hy), None, local))

    e2e_step()
    t0 = time.perf_counter()
    for _ in range(max(1, args.e2e_steps)):
        e2e_step()
    e2e_s = torch.tensor([(time.perf_counter() - t0) / max(1, args.e2e_steps)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        v, info = cpu_reference(wl, threads, target_s=8.0, kind="reference")
        cpu = {"value": v, "unit": "TFLOP/s", "cores": info["cores"], "kind": info["kind"],
               "sample": info["sample"] + " (the grid's largest cell, 16x16x256->1024)",
               "ms_full_layer_extrapolated": info["ms_full_layer_extrapolated"]}
    if rank == 0:
        out = {
            "metric": "RI-conv layer effective TFLOP/s", "value": value, "unit": "TFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "mixed: " + ", ".join(sorted({arith_dtype(c["desc"].kernel_name()) for c in cells})),
            "data": "synthetic (uniform[-1,1) inputs, uniform/sqrt(Cin*K^2) weights, random init)",
            "config": {"workload": wl[-1], "global_batch": n * world, "n_per_gpu": n, "cells": len(cells),
                       "sizes": list(C2_SIZES), "c_in": list(C2_CINS), "c_out": list(C2_COUTS), "k": 3,
                       "group": "single", "orientations": 1, "parallelism": f"replicas dp{world}"},
            "precision": args.precision, "l2": "flushed between timed iterations (512 MB write)",
            "per_rank_ms": [round(t.item() / args.steps, 4) for t in per_rank],
            "timing": "max over ranks of each rank's CUDA-event time of one CUDA-graph replay of the grid",
            "roofline": {"bound": "tensor" if tc else "fp32-simt", "kernel": big["desc"].kernel_name(),
                         "cell": "16x16x256->1024", "achieved": achieved,
                         "peak": tpeak if tc else FFMA_PEAK, "unit": "TFLOP/s",
                         "frac": (achieved / (tpeak if tc else FFMA_PEAK)) if achieved else None,
                         "kernel_ms": kernel_ms, "traffic": None,
                         "peak_source": f"{src} dense bf16 (MEASURED_PEAKS.json)" if tc else PEAKS_SRC},
            "clocks": clk.summary(),
            "e2e": {"value": eff * world / e2e_s.item() / 1e12, "unit": "TFLOP/s",
                    "h2d_bytes_per_step": int(sum(h[1].numel() * 4 + h[2].numel() * 4 for h in hbuf)),
                    "d2h_bytes_per_step": int(sum(h[3].numel() * 4 for h in hbuf)),
                    "ms_per_step": e2e_s.item() * 1e3, "path": "rc_ri_conv_forward_host per cell (C-ABI)"},
            "gpu_launches": args.steps * sum(2 if c["desc"].kernel_name().startswith("tc_") else 1 for c in cells),
            "cpu_baseline": cpu,
            "cells_vs_cudnn": {"columns": ["size", "c_in", "c_out", "kernel", "ours_ms", "cudnn_fp32_ms",
                                           "cudnn_tf32_ms", "speedup_vs_fp32", "err_vs_cudnn"],
                               "rows": rows, "cells_at_or_above_cudnn_fp32": wins},
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="auto", choices=["fp32", "bf16x3", "bf16", "auto"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cudnn", action="store_true", help="skip the cuDNN context measurement")
    ap.add_argument("--no-backward", action="store_true", help="skip the layer-backward context measurement")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        if args.workload == "c5":
            return run_stack_reference(args, wl)
        return run_reference(args, wl)
    if args.workload == "c5":
        return run_stack(args, wl)
    if args.workload == "c2":
        return run_grid(args, wl)

    import torch
    import torch.distributed as dist
    import paper_2512_08888_b200 as P
    from paper_2512_08888_b200 import _lib

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines on stderr (rank check)
        dist.init_process_group("nccl", device_id=dev)
    n, cin, h, w, cout, k, g, R, pool, pg, label = wl
    strong = args.workload in STRONG
    n_global = n if strong else n * world
    if strong:  # this rank's contiguous shard of the global batch (rc_shard_range)
        b0, b1 = P.shard_range(n, world, rank)
        n = b1 - b0
    desc = P.Desc(n, cin, h, w, cout, k, g, R, pool, pg, "scatter", args.precision)
    gen = torch.Generator(device=dev).manual_seed(1234)  # same weights on every rank
    s = 1 / np.sqrt(cin * k * k)
    fx = ((torch.rand((cout, cin, k, k), generator=gen, device=dev) * 2 - 1) * s).contiguous()
    fy = ((torch.rand((cout, cin, k, k), generator=gen, device=dev) * 2 - 1) * s).contiguous()
    bias = (torch.rand(cout, generator=gen, device=dev) * 0.2 - 0.1).contiguous()
    gen.manual_seed(99 + rank)  # each rank its own shard of images
    x = (torch.rand((n, cin, h, w), generator=gen, device=dev) * 2 - 1).contiguous()
    bank = P.bank_precompute(desc, fx, fy)
    ro = desc.out_orientations
    y = torch.empty((n, cout, ro, h, w), device=dev)
    am = torch.empty((n, cout, ro, h, w), dtype=torch.uint8, device=dev) if desc.has_argmax else None
    flush = torch.empty(512 * 1024 * 1024 // 4, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream(dev)

    def step():
        P.ri_conv_forward(desc, x, bank, bias, out=y, argmax=am)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    L = _lib.lib()
    L.rc_profile_enable(1)  # CUDA events around the main kernel of every launch (same stream)
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))  # L2 flush between timed iterations (untimed)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        clk.sample()  # the queued steps are still running on the GPU
        torch.cuda.synchronize()
    L.rc_profile_enable(0)
    kms = (C.c_float * args.steps)()
    nk = L.rc_profile_collect(kms, args.steps)
    kernel_ms = statistics.mean(kms[:nk]) if nk > 0 else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times = [a.elapsed_time(b) for a, b in ev]  # ms, on the launching stream
    tot = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
    per_rank = [tot.clone() for _ in range(world)]
    if world > 1:
        dist.all_gather(per_rank, tot)
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    per_rank_ms = [round(t.item() / args.steps, 4) for t in per_rank]
    ms = tot.item() / args.steps
    eff_total = 2 * n_global * h * w * k * k * cin * cout * R  # all ranks' images
    value = eff_total / (ms * 1e-3) / 1e12
    alg = desc.alg_flops()
    achieved = alg / ((kernel_ms or statistics.mean(times)) * 1e-3) / 1e12
    tpeak, hbm, src = peaks()
    tc = desc.kernel_name().startswith("tc_")
    passes = 3 if tc and args.precision in ("auto", "bf16x3") else 1

    # e2e through the C-ABI host entry point: pinned host buffers, H2D + D2H timed
    hx = torch.empty((n, cin, h, w), dtype=torch.float32, pin_memory=True)
    hx.copy_(x)
    hfx, hfy, hb = (t.cpu().pin_memory() for t in (fx, fy, bias))
    hy = torch.empty((n, cout, ro, h, w), dtype=torch.float32, pin_memory=True)
    ha = torch.empty((n, cout, ro, h, w), dtype=torch.uint8, pin_memory=True) if am is not None else None
    cd = desc.c()
    pp = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None
    _lib.check(L.rc_ri_conv_forward_host(C.byref(cd), pp(hx), pp(hfx), pp(hfy), pp(hb), pp(hy), pp(ha), local))
    if world > 1:
        dist.barrier()
    e2e_t = []
    for _ in range(max(1, args.e2e_steps)):
        t0 = time.perf_counter()
        _lib.check(L.rc_ri_conv_forward_host(C.byref(cd), pp(hx), pp(hfx), pp(hfy), pp(hb), pp(hy), pp(ha), local))
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = torch.tensor([statistics.mean(e2e_t)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_val = eff_total / e2e_s.item() / 1e12
    h2d = hx.numel() * 4 + hfx.numel() * 4 * 2 + hb.numel() * 4
    d2h = hy.numel() * 4 + (ha.numel() if ha is not None else 0)
    # parity spot check of the timed output (image 0) against the e2e path
    ok = torch.equal(y[0].cpu(), hy[0]) if rank == 0 else True

    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        tr = json.load(open(prof)).get(f"{args.workload}:{desc.kernel_name()}")
        traffic = tr
    cudnn_ctx = None
    if rank == 0 and world == 1 and not args.no_cudnn:
        cudnn_ctx = cudnn_context(P, desc, x, fx, fy, ms, args)
    bwd = None
    if rank == 0 and world == 1 and not args.no_backward:
        bwd = backward_context(P, desc, x, bank, y, am)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        v, info = cpu_reference(wl, threads, target_s=8.0, kind="reference")
        cpu = {"value": v, "unit": "TFLOP/s", "cores": info["cores"], "kind": info["kind"],
               "sample": info["sample"], "ms_full_layer_extrapolated": info["ms_full_layer_extrapolated"]}
        if R > 1:  # second row: the paper's reuse algorithm on the CPU (same sample size)
            vp, ip = cpu_reference(wl, threads, target_s=0.0, kind="port", m0=info["images"])
            cpu["port_reuse"] = {"value": vp, "unit": "TFLOP/s", "cores": ip["cores"], "kind": ip["kind"],
                                 "sample": ip["sample"],
                                 "ms_full_layer_extrapolated": ip["ms_full_layer_extrapolated"]}
    if rank == 0:
        out = {
            "metric": "RI-conv layer effective TFLOP/s", "value": value, "unit": "TFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
            "dtype": arith_dtype(desc.kernel_name()),
            "data": "synthetic (uniform[-1,1) inputs, uniform/sqrt(Cin*K^2) weights, random init)",
            "config": workload_config(args, wl, world),
            "precision": args.precision, "kernel": desc.kernel_name(),
            "l2": "flushed between timed iterations (512 MB write)",
            "alg_tflops": achieved * 1.0, "eff_tflops_per_gpu": value / world,
            "per_rank_ms": per_rank_ms, "timing": "max over ranks of each rank's CUDA-event step time",
            "roofline": {"bound": "tensor" if tc else "fp32-simt", "kernel": desc.kernel_name(),
                         "achieved": achieved, "peak": tpeak if tc else FFMA_PEAK, "unit": "TFLOP/s",
                         "frac": achieved / (tpeak if tc else FFMA_PEAK), "traffic": traffic,
                         "kernel_ms": kernel_ms, "step_ms": ms,
                         "peak_source": (f"{src} dense bf16 (MEASURED_PEAKS.json)" if tc else
                                         f"measured FP32 FFMA peak ({PEAKS_SRC})"),
                         "other_measured_peaks": PROBED_PEAKS,
                         "mma_passes": passes,
                         "frac_of_pass_ceiling": achieved * passes / tpeak if tc else None,
                         "smem": smem_roofline(desc, kernel_ms),
                         "note": "achieved = algorithmic FLOPs 2*N*H*W*K^2*Cin*Cout*B per launch / the main "
                                 "kernel's CUDA-event time (rc_profile_*; operand packing excluded). bf16x3 "
                                 "issues 3 bf16 MMAs per FP32-class product: frac_of_pass_ceiling = "
                                 "achieved*passes/peak"},
            "clocks": clk.summary(),
            "e2e": {"value": e2e_val, "unit": "TFLOP/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_s.item() * 1e3,
                    "path": "rc_ri_conv_forward_host (C-ABI, pinned host buffers)"},
            "gpu_launches": args.steps * (2 if desc.kernel_name().startswith("tc_") else 1),
            "gpu_launches_note": "per step: tc path = x_pack_kernel + ri_tc_kernel; SIMT = one fused kernel",
            "cpu_baseline": cpu,
            "cudnn_context": cudnn_ctx,
            "backward_context": bwd,
            "timed_output_matches_e2e": bool(ok),
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
