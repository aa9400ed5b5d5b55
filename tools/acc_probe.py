"""Normwise error of the single-orientation tensor-core conv (implicit GEMM) vs float64 as
the reduction length Cin*9 grows (bf16x3 and bf16), with cuDNN FP32 for comparison."""
import os
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_08888_b200 as P  # noqa: E402

torch.backends.cudnn.allow_tf32 = False
for cin in (256, 1024, 4096, 8192):
    for sparse in (False, True):
        g = torch.Generator(device="cuda").manual_seed(cin)
        n, h, w, cout = 2, 16, 16, 256
        x = torch.rand((n, cin, h, w), generator=g, device="cuda") * 2 - 1
        if sparse:  # like the pool-backward gradient: 3 of 4 channel groups zero
            x = x * (torch.rand((n, cin, h, w), generator=g, device="cuda") < 0.25)
        w0 = (torch.rand((cout, cin, 3, 3), generator=g, device="cuda") * 2 - 1) / (cin * 9) ** 0.5
        ref = F.conv2d(x.double(), torch.flip(w0, dims=(2, 3)).double(), padding=1)
        cud = F.conv2d(x, torch.flip(w0, dims=(2, 3)), padding=1)
        row = [f"cin={cin}", f"sparse={sparse}", "cudnn_fp32=%.2e" % ((cud.double() - ref).abs().max() / ref.abs().max())]
        for prec in ("bf16x3", "bf16"):
            d = P.Desc(n, cin, h, w, cout, 3, "single", 1, "none", 1, "scatter", prec)
            bank = P.bank_precompute(d, w0)
            y, _ = P.ri_conv_forward(d, x, bank)
            row.append("%s=%.2e" % (prec, ((y[:, :, 0].double() - ref).abs().max() / ref.abs().max())))
        print(" ".join(row), flush=True)
