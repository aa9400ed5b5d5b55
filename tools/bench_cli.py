"""SPEC bench_cli on B200: the Appendix-A style sweep across dataflow modes.

    python tools/bench_cli.py [--sizes 8 16 32] [--cin 64 256] [--cout 256 1024]
        [--orientations 4] [--modes scatter gather im2col_matmul group_scatter group_gather]
        [--kernel 3] [--batch 32] [--group steer] [--precision auto] [--repeats 20]
        [--warmup 3] [--workers 1] [--seed 0] [--out sweep.csv] [--format csv|md]

Modes (one cell at a time, identical seeded inputs across modes):
  scatter        single-orientation scatter conv, this repo's fused kernel (rc_ri_conv_forward)
  gather         the same conv as gather-"same" -- cuDNN (torch conv2d on the flipped kernel;
                 cuDNN is the paper's baseline; context only, not the product path)
  im2col_matmul  unfold + cuBLAS matmul (context)
  group_scatter  R-orientation RI conv with channel-dot reuse, this repo's kernel, pool none
  group_gather   the same R slices as R separate cuDNN convs on the rotated kernels (the
                 paper's cuDNN RI pipeline; context)
Every cell runs a correctness cross-check (scatter vs gather, group_scatter vs group_gather,
normwise <= 1e-4) BEFORE timing; the exit code is nonzero if any check fails.  wall_ms is
the median device time (CUDA events around CUDA-graph replays, launch overhead excluded).
The CSV header is exactly SPEC's; the markdown table adds the gather/scatter speedup.
"""
from __future__ import annotations

import argparse
import csv
import math
import os
import statistics
import sys

import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

HEADER = ["mode", "input_size", "in_channels", "out_channels", "orientations", "repeats", "wall_ms", "mults",
          "peak_aux_bytes"]
INNER = 5


def time_ms(fn, repeats, warmup):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(max(1, warmup)):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(INNER):
            fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(repeats):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / INNER)
    return statistics.median(ts)


def rotated_kernels(P, desc, w0, w1):
    """All R orientation kernels (orbit-major) from the repo's bank kernel, (R, Cout, Cin, K, K)."""
    return P.rotconv.build_orientation_bank_from(desc, w0, w1)


def cell_seed(args, size, cin, cout):
    """Identical seeds per cell across modes."""
    return args.seed + size * 7919 + cin * 31 + cout


def cell_tensors(size, cin, cout, args, gen):
    """The cell's seeded inputs X (n, cin, size, size) and kernels W0, W1 (cout, cin, k, k)."""
    dev = torch.device("cuda")
    n, k = args.batch, args.kernel
    x = (torch.rand((n, cin, size, size), generator=gen, device=dev) * 2 - 1).contiguous()
    s = 1 / math.sqrt(cin * k * k)
    w0 = ((torch.rand((cout, cin, k, k), generator=gen, device=dev) * 2 - 1) * s).contiguous()
    w1 = ((torch.rand((cout, cin, k, k), generator=gen, device=dev) * 2 - 1) * s).contiguous()
    return x, w0, w1


def run_cell(P, mode, size, cin, cout, args, gen):
    dev = torch.device("cuda")
    n, k, R = args.batch, args.kernel, args.orientations
    x, w0, w1 = cell_tensors(size, cin, cout, args, gen)
    base_mults = n * size * size * k * k * cin * cout
    if mode in ("scatter", "gather", "im2col_matmul"):
        desc = P.Desc(n, cin, size, size, cout, k, "single", 1, "none", 1, "scatter", args.precision)
        bank = P.bank_precompute(desc, w0)
        y = torch.empty((n, cout, 1, size, size), device=dev)
        wf = torch.flip(w0, dims=(2, 3)).contiguous()
        P.ri_conv_forward(desc, x, bank, out=y)
        ref = F.conv2d(x, wf, padding=k // 2)
        err = ((y[:, :, 0] - ref).abs().max() / ref.abs().max()).item()
        if mode == "scatter":
            fn = lambda: P.ri_conv_forward(desc, x, bank, out=y)
            aux = desc.workspace_bytes() + desc.bank_bytes()
        elif mode == "gather":
            fn = lambda: F.conv2d(x, wf, padding=k // 2)
            aux = 0
        else:
            wm = wf.reshape(cout, -1)
            fn = lambda: (wm @ F.unfold(x, k, padding=k // 2)).view(n, cout, size, size)
            aux = n * cin * k * k * size * size * 4
        return base_mults, aux, err, fn, 1
    group = args.group  # p4 needs R = 4, p4m R = 8, steer any multiple of 4
    desc = P.Desc(n, cin, size, size, cout, k, group, R, "none", 1, "scatter", args.precision)
    bank = P.bank_precompute(desc, w0, w1 if group == "steer" else None)
    y = torch.empty((n, cout, R, size, size), device=dev)
    P.ri_conv_forward(desc, x, bank, out=y)
    kern = rotated_kernels(P, desc, w0, w1 if group == "steer" else None)   # (R, Cout, Cin, K, K)
    # slice o = scatter_conv_multi(X, rot^r K_b) = conv2d(X, flip(rot^r K_b)) (convention P1)
    wcat = torch.flip(kern, dims=(3, 4)).reshape(R * cout, cin, k, k).contiguous()
    ref = F.conv2d(x, wcat, padding=k // 2).view(n, R, cout, size, size).transpose(1, 2)
    err = ((y - ref).abs().max() / ref.abs().max()).item()
    if mode == "group_scatter":
        return base_mults * desc.num_bases, desc.workspace_bytes() + desc.bank_bytes(), err, \
            (lambda: P.ri_conv_forward(desc, x, bank, out=y)), R
    return base_mults * R, 0, err, (lambda: F.conv2d(x, wcat, padding=k // 2)), R


def parse_args(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--sizes", type=int, nargs="+", default=[8, 16, 32])
    ap.add_argument("--cin", type=int, nargs="+", default=[64, 256])
    ap.add_argument("--cout", type=int, nargs="+", default=[256, 1024])
    ap.add_argument("--orientations", type=int, default=8)
    ap.add_argument("--modes", nargs="+", default=["scatter", "gather", "im2col_matmul", "group_scatter",
                                                    "group_gather"])
    ap.add_argument("--kernel", type=int, default=3)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--group", default="steer", choices=["p4", "p4m", "steer"])
    ap.add_argument("--precision", default="auto", choices=["auto", "fp32", "bf16x3", "bf16"])
    ap.add_argument("--repeats", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workers", type=int, default=1, help="accepted for SPEC parity; the GPU ignores it")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--format", default="csv", choices=["csv", "md"])
    return ap.parse_args(argv)


def main(argv=None):
    args = parse_args(argv)
    import paper_2512_08888_b200 as P
    torch.backends.cudnn.benchmark = True
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    recs, failed = [], 0
    for size in args.sizes:
        for cin in args.cin:
            for cout in args.cout:
                for mode in args.modes:
                    if args.kernel > size:
                        print(f"skip {mode} {size}x{size}: kernel > input", file=sys.stderr)
                        continue
                    gen = torch.Generator(device="cuda").manual_seed(cell_seed(args, size, cin, cout))
                    mults, aux, err, fn, R = run_cell(P, mode, size, cin, cout, args, gen)
                    if not err <= 1e-4:
                        failed += 1
                        print(f"CROSS-CHECK FAILED {mode} {size} {cin} {cout}: {err:.3e}", file=sys.stderr)
                        continue
                    ms = time_ms(fn, args.repeats, args.warmup)
                    recs.append({"mode": mode, "input_size": size, "in_channels": cin, "out_channels": cout,
                                 "orientations": R, "repeats": args.repeats, "wall_ms": round(ms, 5),
                                 "mults": mults, "peak_aux_bytes": aux})
                    print(",".join(str(recs[-1][h]) for h in HEADER), flush=True)
    if not recs:
        print("no records", file=sys.stderr)
        return 1
    if args.out:
        if args.format == "csv":
            with open(args.out, "w", newline="") as f:
                w = csv.DictWriter(f, fieldnames=HEADER)
                w.writeheader()
                w.writerows(recs)
        else:
            with open(args.out, "w") as f:
                f.write("| " + " | ".join(HEADER) + " | speedup (gather or group_gather ms / this ms) |\n")
                f.write("|" + "---|" * (len(HEADER) + 1) + "\n")
                for r in recs:
                    base = "group_gather" if r["mode"].startswith("group") else "gather"
                    ref = [q for q in recs if q["mode"] == base and all(
                        q[c] == r[c] for c in ("input_size", "in_channels", "out_channels"))]
                    sp = f"{ref[0]['wall_ms'] / r['wall_ms']:.2f}" if ref else ""
                    f.write("| " + " | ".join(str(r[h]) for h in HEADER) + f" | {sp} |\n")
    return 1 if failed else 0


if __name__ == "__main__":
    sys.exit(main())
