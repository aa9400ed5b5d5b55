"""Backward of the fused RI layer (SPEC backward module) against autograd of a
float64 PyTorch restatement of the forward (test infrastructure: conv2d on the rotated,
flipped slice kernels of convention P1, then pooling / bias / ReLU).

The reference routes max-pool gradients through THIS library's argmax map (the forward's
own tie rule, SPEC "Max-pool gradient at ties follows the forward tie rule"), so near-ties
between the FP32 forward and the float64 restatement cannot mis-route a gradient.

Tolerances, normwise max|d - d_ref| / max|d_ref| per gradient:
  fp32 (CUDA-core forward; backward input pass on the same kernels, weights FP32 SGEMM) 1e-5
  bf16x3 (tensor-core input pass)                                                        1e-4
Plus the SPEC examples: zero upstream -> zero gradients; pool_backward partition of unity.
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu


TOL_LARGE = 1e-4  # SPEC 32-bit tolerance, also at 73728-term reductions (segmented TMEM accumulation)


def ref_forward(x, w0, w1, bias, desc, am=None):
    """float64 forward of convention P1 (slice (b, r) = scatter_conv_multi(X, rot90^r K_b))."""
    k = desc.k
    if desc.group in ("single", "p4"):
        bases = [w0]
    elif desc.group == "p4m":
        bases = [w0, torch.flip(w0, dims=[-1])]  # mirror_plane, tensor.hpp:363-370
    else:
        nb = desc.orientations // 4
        bases = [math.sin(2 * math.pi * b / desc.orientations) * w0 + math.cos(2 * math.pi * b / desc.orientations) * w1
                 for b in range(nb)]
    rpb = 1 if desc.group == "single" else 4
    slices = []
    for kb in bases:
        for r in range(rpb):
            g = torch.rot90(kb, r, dims=(-2, -1))  # rot90_plane^r, tensor.hpp:348-360
            f = torch.flip(g, dims=(-2, -1)) if desc.convention == "scatter" else g
            slices.append(F.conv2d(x, f, padding=k // 2))
    fstack = torch.stack(slices, dim=2)  # (N, Cout, R, H, W)
    n, co, R, h, w = fstack.shape
    if desc.pool == "none":
        y = fstack
    elif desc.pool == "avg":
        y = fstack.mean(dim=2, keepdim=True)
    else:  # max / subgroup: select through the library's argmax (its tie rule)
        g = R if desc.pool == "max" else desc.pool_group
        blocks = fstack.view(n, co, R // g, g, h, w)
        y = torch.gather(blocks, 3, am.long().view(n, co, R // g, 1, h, w)).squeeze(3)
    if bias is not None:
        y = y + bias.view(1, -1, 1, 1, 1)
    if desc.activation == "relu":
        y = torch.relu(y)
    return y


CASES = [
    # (n, cin, h, w, cout, group, R, pool, g, convention, activation)
    (2, 16, 16, 16, 32, "steer", 8, "subgroup", 4, "scatter", "relu"),
    (2, 64, 16, 16, 128, "p4m", 8, "max", 8, "scatter", "none"),
    (1, 32, 8, 8, 64, "p4", 4, "avg", 4, "raw", "none"),
    (2, 24, 32, 32, 40, "single", 1, "none", 1, "scatter", "relu"),
    (1, 16, 12, 20, 24, "steer", 16, "subgroup", 4, "scatter", "none"),
]


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-5), ("bf16x3", 1e-4)])
@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(map(str, c)))
def test_backward_vs_float64_autograd(dev, case, precision, tol):
    import paper_2512_08888_b200 as P
    n, cin, h, w, cout, g, R, pool, pg, conv, act = case
    prec = precision
    desc = P.Desc(n, cin, h, w, cout, 3, g, R, pool, pg, conv, prec, act)
    if prec == "bf16x3" and not (desc.kernel_name() or "").startswith("tc_"):
        desc = P.Desc(n, cin, h, w, cout, 3, g, R, pool, pg, conv, "fp32", act)
    gen = torch.Generator(device=dev).manual_seed(7)
    x = torch.rand((n, cin, h, w), generator=gen, device=dev) * 2 - 1
    s = 1 / math.sqrt(cin * 9)
    w0 = (torch.rand((cout, cin, 3, 3), generator=gen, device=dev) * 2 - 1) * s
    w1 = (torch.rand((cout, cin, 3, 3), generator=gen, device=dev) * 2 - 1) * s if g == "steer" else None
    bias = torch.rand(cout, generator=gen, device=dev) * 0.2 - 0.1
    bank = P.bank_precompute(desc, w0, w1)
    y, am = P.ri_conv_forward(desc, x, bank, bias)
    m = torch.rand(y.shape, generator=gen, device=dev) * 2 - 1  # loss = sum(y * m)
    dx, dw0, dw1, db = P.ri_conv_backward(desc, x, bank, m, y, am)
    # float64 reference through autograd
    xd = x.double().requires_grad_()
    w0d = w0.double().requires_grad_()
    w1d = w1.double().requires_grad_() if w1 is not None else None
    bd = bias.double().requires_grad_()
    yref = ref_forward(xd, w0d, w1d, bd, desc, am)
    assert torch.allclose(y.double(), yref, atol=5e-3 * yref.abs().max().item())
    (yref * m.double()).sum().backward()
    rel = lambda a, b: ((a.double() - b).abs().max() / b.abs().max()).item()
    assert rel(dx, xd.grad) <= tol, ("dx", rel(dx, xd.grad))
    assert rel(dw0, w0d.grad) <= tol, ("dw0", rel(dw0, w0d.grad))
    if w1 is not None:
        assert rel(dw1, w1d.grad) <= tol, ("dw1", rel(dw1, w1d.grad))
    assert rel(db, bd.grad) <= 1e-5, ("db", rel(db, bd.grad))


@pytest.mark.parametrize("case", [(2, 256, 16, 16, 1024, "steer", 8, "subgroup", 4, "scatter", "none"),
                                  (3, 64, 32, 32, 128, "p4m", 8, "max", 8, "scatter", "relu"),
                                  (256, 32, 16, 16, 32, "p4", 4, "avg", 4, "scatter", "none")],
                         ids=lambda c: "-".join(map(str, c)))
def test_backward_large_tensor_core(dev, case):
    """The C3 layer shape (tensor-core weight gradient without K splits: 512 work items) and a
    32x32 p4m layer, bf16x3, against float64 autograd: normwise <= 1e-4 per gradient."""
    import paper_2512_08888_b200 as P
    n, cin, h, w, cout, g, R, pool, pg, conv, act = case
    desc = P.Desc(n, cin, h, w, cout, 3, g, R, pool, pg, conv, "bf16x3", act)
    gen = torch.Generator(device=dev).manual_seed(17)
    x = torch.rand((n, cin, h, w), generator=gen, device=dev) * 2 - 1
    s = 1 / math.sqrt(cin * 9)
    w0 = (torch.rand((cout, cin, 3, 3), generator=gen, device=dev) * 2 - 1) * s
    w1 = (torch.rand((cout, cin, 3, 3), generator=gen, device=dev) * 2 - 1) * s if g == "steer" else None
    bias = torch.rand(cout, generator=gen, device=dev) * 0.2 - 0.1
    bank = P.bank_precompute(desc, w0, w1)
    y, am = P.ri_conv_forward(desc, x, bank, bias)
    m = torch.rand(y.shape, generator=gen, device=dev) * 2 - 1
    dx, dw0, dw1, db = P.ri_conv_backward(desc, x, bank, m, y, am)
    xd = x.double().requires_grad_()
    w0d = w0.double().requires_grad_()
    w1d = w1.double().requires_grad_() if w1 is not None else None
    bd = bias.double().requires_grad_()
    yref = ref_forward(xd, w0d, w1d, bd, desc, am)
    (yref * m.double()).sum().backward()
    rel = lambda a, b: ((a.double() - b).abs().max() / b.abs().max()).item()
    errs = {"dx": rel(dx, xd.grad), "dw0": rel(dw0, w0d.grad), "db": rel(db, bd.grad)}
    if w1 is not None:
        errs["dw1"] = rel(dw1, w1d.grad)
    print("normwise errors", errs)
    # fan-in of these reductions: dx 9*Cout*R (73728 at the C3 shape), dW N*H*W (K of the
    # tensor-core accumulators); the implicit GEMM segments long reductions (ri_igemm.cu)
    assert errs["dx"] <= TOL_LARGE and errs["dw0"] <= TOL_LARGE and errs.get("dw1", 0) <= TOL_LARGE, errs
    assert errs["db"] <= 1e-5, errs


def test_weight_gradient_many_k_splits(dev):
    """A thin layer over a large batch: 1 m-tile x 1 ci-chunk, so the tensor-core weight
    gradient splits K over ~143 work items (no split may be empty) and reduces them."""
    import paper_2512_08888_b200 as P
    n, cin, h, w, cout = 480, 8, 16, 16, 16
    desc = P.Desc(n, cin, h, w, cout, 3, "p4", 4, "avg", 4, "scatter", "bf16x3")
    gen = torch.Generator(device=dev).manual_seed(23)
    x = torch.rand((n, cin, h, w), generator=gen, device=dev) * 2 - 1
    w0 = (torch.rand((cout, cin, 3, 3), generator=gen, device=dev) * 2 - 1) / math.sqrt(cin * 9)
    bank = P.bank_precompute(desc, w0)
    y, am = P.ri_conv_forward(desc, x, bank)
    m = torch.rand(y.shape, generator=gen, device=dev) * 2 - 1
    _, dw0, _, _ = P.ri_conv_backward(desc, x, bank, m, y, am, need_input=False, need_bias=False)
    w0d = w0.double().requires_grad_()
    (ref_forward(x.double(), w0d, None, None, desc, am) * m.double()).sum().backward()
    err = ((dw0.double() - w0d.grad).abs().max() / w0d.grad.abs().max()).item()
    assert err <= 1e-4, err


def test_empty_batch_zero_parameter_gradients(dev):
    import paper_2512_08888_b200 as P
    desc = P.Desc(0, 16, 8, 8, 32, 3, "steer", 8, "subgroup", 4, "scatter", "auto")
    x = torch.empty((0, 16, 8, 8), device=dev)
    w0 = torch.rand((32, 16, 3, 3), device=dev)
    w1 = torch.rand((32, 16, 3, 3), device=dev)
    bank = P.bank_precompute(desc, w0, w1)
    gy = torch.empty((0, 32, 2, 8, 8), device=dev)
    am = torch.empty(gy.shape, dtype=torch.uint8, device=dev)
    _, dw0, dw1, db = P.ri_conv_backward(desc, x, bank, gy, None, am)
    assert not dw0.any() and not dw1.any() and not db.any()


def test_autograd_function_and_zero_upstream(dev):
    import paper_2512_08888_b200 as P
    desc = P.Desc(2, 16, 16, 16, 32, 3, "steer", 8, "subgroup", 4, "scatter", "auto", "relu")
    gen = torch.Generator(device=dev).manual_seed(3)
    x = (torch.rand((2, 16, 16, 16), generator=gen, device=dev) * 2 - 1).requires_grad_()
    w0 = (torch.rand((32, 16, 3, 3), generator=gen, device=dev) * 0.2 - 0.1).requires_grad_()
    w1 = (torch.rand((32, 16, 3, 3), generator=gen, device=dev) * 0.2 - 0.1).requires_grad_()
    b = torch.zeros(32, device=dev, requires_grad=True)
    y = P.rotconv.RIConvFunction.apply(x, w0, w1, b, desc)
    (y * 0).sum().backward()  # SPEC: zero upstream -> zero gradients
    assert not x.grad.any() and not w0.grad.any() and not w1.grad.any() and not b.grad.any()
    x.grad = None
    y = P.rotconv.RIConvFunction.apply(x, w0, w1, b, desc)
    y.sum().backward()
    assert x.grad is not None and torch.isfinite(x.grad).all() and w1.grad.abs().sum() > 0


def test_pool_backward_partition_of_unity(dev):
    """sum over slices of the pool gradient equals G (avg and max)."""
    import paper_2512_08888_b200 as P
    for pool, g in (("avg", 4), ("max", 8), ("subgroup", 4)):
        desc = P.Desc(1, 8, 8, 8, 16, 3, "p4m", 8, pool, g, "scatter", "fp32")
        gen = torch.Generator(device=dev).manual_seed(1)
        x = torch.rand((1, 8, 8, 8), generator=gen, device=dev)
        w0 = torch.rand((16, 8, 3, 3), generator=gen, device=dev)
        bank = P.bank_precompute(desc, w0)
        y, am = P.ri_conv_forward(desc, x, bank)
        gy = torch.rand(y.shape, generator=gen, device=dev)
        _, _, _, db = P.ri_conv_backward(desc, x, bank, gy, y, am, need_input=False, need_weight=False)
        assert torch.allclose(db, gy.sum(dim=(0, 2, 3, 4)), rtol=1e-5)
