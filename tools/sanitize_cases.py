"""Small launches of every product kernel family for compute-sanitizer (memcheck / racecheck /
synccheck): the tcgen05 band kernel (carry bands on 16-wide images and strips, 8x8 / 4x4 images,
streamed X), the implicit GEMM, the direct small-Cin kernel, the FP32 CUDA-core kernels, the generic kernel, and the backward (pool / input /
tcgen05 weight gradient).  Prints one line per case; exits non-zero on a CUDA error.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_08888_b200 as P  # noqa: E402

CASES = [
    # (n, cin, h, w, cout, group, R, pool, g, precision)
    (3, 64, 16, 16, 256, "steer", 8, "subgroup", 4, "bf16x3"),   # w16 bands, 2 co tiles
    (2, 32, 8, 48, 128, "p4m", 8, "max", 8, "bf16x3"),           # strips
    (2, 16, 8, 8, 128, "p4", 4, "avg", 4, "bf16"),               # 8x8 images
    (5, 32, 4, 4, 128, "p4m", 8, "subgroup", 4, "bf16x3"),       # 4x4 images, ragged group
    (1, 576, 6, 32, 130, "p4", 4, "max", 4, "bf16x3"),           # streamed X (Cin > 512)
    (2, 64, 12, 20, 96, "single", 1, "none", 1, "bf16x3"),       # implicit GEMM
    (4, 6, 8, 8, 40, "single", 1, "max", 1, "auto"),              # direct FP32 small-Cin kernel
    (2, 5, 16, 16, 7, "steer", 8, "subgroup", 4, "fp32"),        # SIMT FP32
    (2, 3, 7, 5, 4, "p4", 4, "max", 4, "fp32"),                  # generic (K = 5 below)
]


def main():
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    for n, cin, h, w, cout, grp, R, pool, pg, prec in CASES:
        k = 5 if (h, w) == (7, 5) else 3
        d = P.Desc(n, cin, h, w, cout, k, grp, R, pool, pg, "scatter", prec)
        x = torch.rand((n, cin, h, w), generator=g, device=dev) * 2 - 1
        w0 = torch.rand((cout, cin, k, k), generator=g, device=dev) * 0.1
        w1 = torch.rand((cout, cin, k, k), generator=g, device=dev) * 0.1 if grp == "steer" else None
        bias = torch.rand(cout, generator=g, device=dev)
        bank = P.bank_precompute(d, w0, w1)
        y, a = P.ri_conv_forward(d, x, bank, bias)
        torch.cuda.synchronize()
        line = f"fwd {d.kernel_name():20s} ok"
        if k == 3 and h % 2 == 0 and prec != "fp32":
            gy = torch.rand(y.shape, generator=g, device=dev)
            P.ri_conv_backward(d, x, bank, gy, y, a)
            torch.cuda.synchronize()
            line += " | bwd ok"
        print(line, flush=True)
    print("sanitize cases done")


if __name__ == "__main__":
    main()
