"""Where the band kernel's MMA warp waits (RC_TC_ABLATE=10 instrumentation; the clock64 patch
for ri_tc.cu is not in the tree, see profiles/r01/regsplit_ab.txt):
per CTA, total cycles of the MMA warp and the cycles spent waiting for a free TMEM D buffer
(epilogue), for the X band (TMA) and for a weight stage (TMA).  Outputs are overwritten.

    RC_TC_ABLATE=10 python tools/tc_wait_profile.py N CIN H W COUT GROUP R POOL G [precision]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_08888_b200 as P  # noqa: E402

a = sys.argv[1:]
n, cin, h, w, cout = map(int, a[:5])
group, R, pool, g = a[5], int(a[6]), a[7], int(a[8])
prec = a[9] if len(a) > 9 else "auto"
desc = P.Desc(n, cin, h, w, cout, 3, group, R, pool, g, "scatter", prec)
x = torch.rand((n, cin, h, w), device="cuda") * 2 - 1
w0 = torch.rand((cout, cin, 3, 3), device="cuda") * 0.1
w1 = torch.rand((cout, cin, 3, 3), device="cuda") * 0.1 if group == "steer" else None
bank = P.bank_precompute(desc, w0, w1)
for _ in range(3):
    y, _ = P.ri_conv_forward(desc, x, bank)
torch.cuda.synchronize()
v = y.flatten()[: 148 * 4].view(148, 4).double().cpu()
tot, d, xw, ww = v[:, 0], v[:, 1], v[:, 2], v[:, 3]
print(desc.kernel_name(), "MMA-warp cycles per CTA: mean %.3g" % tot.mean().item())
for name, c in (("wait D buffer (epilogue)", d), ("wait X band (TMA)", xw), ("wait W stage (TMA)", ww)):
    print("  %-26s %5.1f%% of the MMA warp's time (max CTA %.1f%%)" % (name, 100 * (c / tot).mean().item(),
                                                                        100 * (c / tot).max().item()))
print("  %-26s %5.1f%%" % ("issuing / other", 100 * (1 - (d + xw + ww) / tot).mean().item()))
