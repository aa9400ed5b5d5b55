"""Time forward and backward (input / weight / all) of one RI layer on the GPU.

    python tools/bwd_probe.py N CIN H W COUT GROUP R POOL G [precision] [activation]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_08888_b200 as P  # noqa: E402


def timed(fn, iters=3):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / iters


a = sys.argv[1:]
n, cin, h, w, cout = map(int, a[:5])
group, R, pool, g = a[5], int(a[6]), a[7], int(a[8])
prec = a[9] if len(a) > 9 else "auto"
act = a[10] if len(a) > 10 else "none"
desc = P.Desc(n, cin, h, w, cout, 3, group, R, pool, g, "scatter", prec, act)
x = torch.rand((n, cin, h, w), device="cuda") * 2 - 1
w0 = torch.rand((cout, cin, 3, 3), device="cuda") * 0.1
w1 = torch.rand((cout, cin, 3, 3), device="cuda") * 0.1 if group == "steer" else None
bank = P.bank_precompute(desc, w0, w1)
bias = torch.rand(cout, device="cuda")
y, am = P.ri_conv_forward(desc, x, bank, bias)
gy = torch.rand(y.shape, device="cuda")
print("kernel", desc.kernel_name())
print("forward ms %.3f" % timed(lambda: P.ri_conv_forward(desc, x, bank, bias)))
print("backward input-only ms %.3f" % timed(lambda: P.ri_conv_backward(desc, x, bank, gy, y, am, need_weight=False,
                                                                       need_bias=False)))
print("backward weight-only ms %.3f" % timed(lambda: P.ri_conv_backward(desc, x, bank, gy, y, am, need_input=False,
                                                                        need_bias=False)))
print("backward all ms %.3f" % timed(lambda: P.ri_conv_backward(desc, x, bank, gy, y, am)))
