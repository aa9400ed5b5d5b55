"""Single-orientation implicit-GEMM tensor-core path (ri_igemm.cu) vs the CPU oracle.

R = 1 layers (group "single": tiled_scatter_conv semantics, scatter_conv.hpp:333-338, and
the "raw" convention the backward input pass uses) run as 9 row-shifted views of one
zero-padded X tile.  Any H, W (not only the band geometries of the RI kernels) and any Cout.
Tolerances as in test_gpu_tc.py: dyadic inputs are exact in bf16, so bf16 and bf16x3 are
bit-exact; random inputs, normwise max|dy|/max|y|: bf16x3 <= 3e-5, bf16 <= 1e-2.
"""
import numpy as np
import pytest
import torch

from conftest import dyadic

pytestmark = pytest.mark.gpu

TOL = {"bf16x3": 3e-5, "bf16": 1e-2}

CONFIGS = [
    # (n, cin, h, w, cout, convention, pool, activation)
    (2, 64, 16, 16, 256, "scatter", "none", "none"),
    (3, 32, 9, 16, 130, "raw", "max", "none"),
    (2, 128, 32, 32, 128, "scatter", "avg", "relu"),
    (1, 16, 5, 7, 64, "raw", "none", "none"),
    (2, 100, 24, 24, 40, "scatter", "none", "relu"),
    (1, 64, 64, 64, 64, "scatter", "none", "none"),
    (3, 48, 11, 33, 300, "scatter", "none", "none"),
    (5, 256, 8, 12, 96, "raw", "none", "none"),
    (1, 200, 1, 1, 200, "scatter", "none", "none"),
    (2, 24, 3, 70, 33, "scatter", "max", "relu"),
    (2, 1100, 6, 10, 72, "scatter", "max", "relu"),   # 3 accumulation segments (8 ci chunks each)
]


def _desc(P, c, precision):
    n, cin, h, w, cout, conv, pool, act = c
    return P.Desc(n, cin, h, w, cout, 3, "single", 1, pool, 1, conv, precision, act)


def _run(P, desc, x, w0, bias, dev):
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    bank = P.bank_precompute(desc, t(w0))
    y, a = P.ri_conv_forward(desc, t(x), bank, t(bias))
    torch.cuda.synchronize()
    return y.cpu().numpy(), (a.cpu().numpy() if a is not None else None)


def _oracle(O, c, x, w0, bias):
    n, cin, h, w, cout, conv, pool, act = c
    d = O.Desc(n, cin, h, w, cout, 3, "single", 1, pool, 1, conv)
    y, _ = O.ri_forward(d, x, w0, None, bias, nthreads=8)
    if act == "relu":
        y = np.maximum(y, 0)
    return y


@pytest.mark.parametrize("precision", ["bf16", "bf16x3"])
@pytest.mark.parametrize("cfg", CONFIGS, ids=lambda c: "-".join(map(str, c)))
def test_igemm_dyadic_bitexact(O, dev, cfg, precision):
    import paper_2512_08888_b200 as P
    n, cin, h, w, cout = cfg[:5]
    desc = _desc(P, cfg, precision)
    assert desc.kernel_name() == f"tc_igemm_{precision}", desc.kernel_name()
    rng = np.random.default_rng(abs(hash(cfg)) % 2**32)
    x = dyadic(rng, (n, cin, h, w))
    w0 = dyadic(rng, (cout, cin, 3, 3))
    bias = dyadic(rng, cout)
    y_ref = _oracle(O, cfg, x, w0, bias)
    y, a = _run(P, desc, x, w0, bias, dev)
    y = y.reshape(y_ref.shape)
    assert np.array_equal(y, y_ref), f"max|dy| = {np.abs(y - y_ref).max()}"
    if a is not None:
        assert not a.any()  # R = 1: the only orientation


@pytest.mark.parametrize("precision", ["bf16", "bf16x3"])
@pytest.mark.parametrize("cfg", [(2, 128, 64, 64, 64, "scatter", "none", "relu"),
                                 (4, 256, 32, 32, 128, "raw", "none", "none"),
                                 (2, 512, 16, 16, 256, "scatter", "none", "relu")],
                         ids=lambda c: "-".join(map(str, c)))
def test_igemm_random_tolerance(O, dev, cfg, precision):
    """The C5 stack's standard convolutions (one image-size step each)."""
    import paper_2512_08888_b200 as P
    n, cin, h, w, cout = cfg[:5]
    desc = _desc(P, cfg, precision)
    rng = np.random.default_rng(11 + abs(hash(cfg)) % 2**31)
    x = rng.uniform(-1, 1, (n, cin, h, w)).astype(np.float32)
    s = 1 / np.sqrt(cin * 9)
    w0 = rng.uniform(-s, s, (cout, cin, 3, 3)).astype(np.float32)
    bias = rng.uniform(-0.1, 0.1, cout).astype(np.float32)
    y_ref = _oracle(O, cfg, x, w0, bias)
    y, _ = _run(P, desc, x, w0, bias, dev)
    err = np.abs(y.reshape(y_ref.shape).astype(np.float64) - y_ref).max() / np.abs(y_ref).max()
    assert err <= TOL[precision], f"normwise {err:.3e}"


def test_igemm_matches_cudnn_large(dev):
    """A full C5 layer-2 shape at batch 64 against cuDNN FP32 (no TF32): normwise <= 3e-5."""
    import paper_2512_08888_b200 as P
    torch.backends.cudnn.allow_tf32 = False
    g = torch.Generator(device=dev).manual_seed(5)
    n, cin, h, w, cout = 64, 128, 64, 64, 64
    x = torch.rand((n, cin, h, w), generator=g, device=dev) * 2 - 1
    w0 = (torch.rand((cout, cin, 3, 3), generator=g, device=dev) * 2 - 1) / (cin * 9) ** 0.5
    desc = P.Desc(n, cin, h, w, cout, 3, "single", 1, "none", 1, "scatter", "bf16x3")
    bank = P.bank_precompute(desc, w0)
    y, _ = P.ri_conv_forward(desc, x, bank)
    ref = torch.nn.functional.conv2d(x, torch.flip(w0, dims=(2, 3)), padding=1)  # convention P1
    err = ((y[:, :, 0] - ref).abs().max() / ref.abs().max()).item()
    assert err <= 3e-5, err
