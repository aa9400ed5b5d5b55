"""Tensor-core (tcgen05) path parity vs the CPU oracle.

Tolerances, stated per arithmetic:
  * dyadic inputs (k/4) are exact in bf16 (hi part; lo part 0), so both "bf16" and
    "bf16x3" reproduce the oracle bit-for-bit (values and argmax) for p4 / p4m;
  * random inputs, normwise max|dy|/max|y|:  bf16x3 <= 3e-5,  bf16 <= 1e-2.
"""
import numpy as np
import pytest
import torch

from conftest import dyadic

pytestmark = pytest.mark.gpu

TOL = {"bf16x3": 3e-5, "bf16": 1e-2}


def run(P, d, x, w0, w1, bias, precision, dev):
    t = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    desc = P.Desc(d.n, d.c_in, d.h, d.w, d.c_out, d.k, d.group, d.orientations, d.pool, d.pool_group,
                  d.convention, precision)
    assert desc.kernel_name().startswith("tc_"), desc.kernel_name()
    bank = P.bank_precompute(desc, t(w0), t(w1))
    y, a = P.ri_conv_forward(desc, t(x), bank, t(bias))
    torch.cuda.synchronize()
    y = y.cpu().numpy()
    a = a.cpu().numpy() if a is not None else None
    if d.pool in ("avg", "max"):
        y = y[:, :, 0]
        a = a[:, :, 0] if a is not None else None
    return y, a


TC_CONFIGS = [
    # (n, cin, h, cout, group, R, pool, g, convention)
    (2, 64, 16, 128, "p4", 4, "subgroup", 4, "scatter"),
    (3, 16, 16, 128, "p4m", 8, "subgroup", 4, "scatter"),
    (2, 100, 13, 200, "p4m", 8, "max", 8, "scatter"),
    (2, 64, 4, 128, "p4", 4, "none", 4, "scatter"),
    (1, 32, 1, 128, "p4", 4, "avg", 4, "raw"),
    (2, 256, 16, 256, "p4m", 8, "subgroup", 2, "scatter"),
    (2, 48, 9, 130, "p4m", 8, "subgroup", 1, "raw"),
    (2, 64, 16, 128, "p4m", 8, "avg", 4, "scatter"),
    (2, 64, 6, 128, "p4m", 8, "max", 8, "scatter"),  # last band: 3 of 6 band rows in the image
    (1, 64, 2, 128, "p4", 4, "none", 4, "raw"),      # one band, top and bottom rows trimmed
]


@pytest.mark.parametrize("precision", ["bf16", "bf16x3"])
@pytest.mark.parametrize("cfg", TC_CONFIGS, ids=lambda c: "-".join(map(str, c)))
def test_tc_dyadic_bitexact(O, dev, cfg, precision):
    import paper_2512_08888_b200 as P
    n, cin, h, cout, g, R, pool, pg, conv = cfg
    d = O.Desc(n, cin, h, 16, cout, 3, g, R, pool, pg, conv)
    rng = np.random.default_rng(abs(hash(cfg)) % 2**32)
    x = dyadic(rng, (n, cin, h, 16))
    w0 = dyadic(rng, (cout, cin, 3, 3))
    bias = dyadic(rng, cout)
    y_ref, a_ref = O.ri_forward(d, x, w0, None, bias)
    y, a = run(P, d, x, w0, None, bias, precision, dev)
    assert np.array_equal(y, y_ref), f"max|dy| = {np.abs(y - y_ref).max()}"
    if a_ref is not None:
        assert np.array_equal(a, a_ref), f"argmax mismatches {(a != a_ref).sum()}"


@pytest.mark.parametrize("precision", ["bf16", "bf16x3"])
@pytest.mark.parametrize("cfg", [(2, 256, 16, 256, "steer", 8, "subgroup", 4),
                                 (2, 128, 16, 128, "steer", 16, "subgroup", 4),
                                 (2, 64, 11, 128, "steer", 12, "max", 12),
                                 (2, 96, 16, 192, "p4m", 8, "subgroup", 4)],
                         ids=lambda c: "-".join(map(str, c)))
def test_tc_random_tolerance(O, dev, cfg, precision):
    import paper_2512_08888_b200 as P
    n, cin, h, cout, g, R, pool, pg = cfg
    d = O.Desc(n, cin, h, 16, cout, 3, g, R, pool, pg)
    rng = np.random.default_rng(7 + abs(hash(cfg)) % 2**31)
    x = rng.uniform(-1, 1, (n, cin, h, 16)).astype(np.float32)
    s = 1 / np.sqrt(cin * 9)
    w0 = rng.uniform(-s, s, (cout, cin, 3, 3)).astype(np.float32)
    w1 = rng.uniform(-s, s, (cout, cin, 3, 3)).astype(np.float32)
    bias = rng.uniform(-0.1, 0.1, cout).astype(np.float32)
    y_ref, a_ref = O.ri_forward(d, x, w0, w1, bias)
    y, a = run(P, d, x, w0, w1, bias, precision, dev)
    err = np.abs(y.astype(np.float64) - y_ref).max() / np.abs(y_ref).max()
    assert err <= TOL[precision], f"normwise {err:.3e}"
    if precision == "bf16x3" and a_ref is not None:
        dn = O.Desc(n, cin, h, 16, cout, 3, g, R, "none")
        f, _ = O.ri_forward(dn, x, w0, w1)
        gg = R if pool == "max" else pg
        blk = np.sort(f.reshape(n, cout, R // gg, gg, h, 16), axis=3)
        gap = blk[:, :, :, -1] - blk[:, :, :, -2]
        if pool == "max":
            gap = gap[:, :, 0]
        safe = gap > 1e-3 * np.abs(y_ref).max()
        assert np.array_equal(a[safe], a_ref[safe])


TC32_CONFIGS = [
    # (n, cin, h, cout, group, R, pool, g, convention) at W = 32
    (2, 64, 32, 128, "p4", 4, "subgroup", 4, "scatter"),
    (2, 128, 7, 256, "p4m", 8, "max", 8, "scatter"),
    (1, 32, 3, 130, "p4m", 8, "subgroup", 2, "raw"),
    (2, 64, 32, 128, "p4", 4, "none", 4, "scatter"),
    (1, 48, 5, 128, "p4m", 8, "avg", 4, "scatter"),
]


@pytest.mark.parametrize("rows32", ["0", "1"])  # W=32 as 4x16 strips (default) or 2-row bands
@pytest.mark.parametrize("precision", ["bf16", "bf16x3"])
@pytest.mark.parametrize("cfg", TC32_CONFIGS, ids=lambda c: "-".join(map(str, c)))
def test_tc_w32_dyadic_bitexact(O, dev, cfg, precision, rows32, monkeypatch):
    monkeypatch.setenv("RC_TC_ROWS32", rows32)
    import paper_2512_08888_b200 as P
    n, cin, h, cout, g, R, pool, pg, conv = cfg
    d = O.Desc(n, cin, h, 32, cout, 3, g, R, pool, pg, conv)
    rng = np.random.default_rng(abs(hash(cfg)) % 2**32)
    x = dyadic(rng, (n, cin, h, 32))
    w0 = dyadic(rng, (cout, cin, 3, 3))
    bias = dyadic(rng, cout)
    y_ref, a_ref = O.ri_forward(d, x, w0, None, bias)
    y, a = run(P, d, x, w0, None, bias, precision, dev)
    assert np.array_equal(y, y_ref), f"max|dy| = {np.abs(y - y_ref).max()}"
    if a_ref is not None:
        assert np.array_equal(a, a_ref), f"argmax mismatches {(a != a_ref).sum()}"


@pytest.mark.parametrize("precision", ["bf16", "bf16x3"])
def test_tc_w32_c4_shape_random(O, dev, precision):
    """C4 layer shape (32x32, 128 -> 512, steer R=16, subgroup-4) on 2 images vs the oracle."""
    import paper_2512_08888_b200 as P
    n, cin, h, cout = 2, 128, 32, 512
    d = O.Desc(n, cin, h, 32, cout, 3, "steer", 16, "subgroup", 4)
    rng = np.random.default_rng(44)
    x = rng.uniform(-1, 1, (n, cin, h, 32)).astype(np.float32)
    s = 1 / np.sqrt(cin * 9)
    w0 = rng.uniform(-s, s, (cout, cin, 3, 3)).astype(np.float32)
    w1 = rng.uniform(-s, s, (cout, cin, 3, 3)).astype(np.float32)
    bias = rng.uniform(-0.1, 0.1, cout).astype(np.float32)
    y_ref, a_ref = O.ri_forward(d, x, w0, w1, bias, nthreads=8)
    y, a = run(P, d, x, w0, w1, bias, precision, dev)
    err = np.abs(y.astype(np.float64) - y_ref).max() / np.abs(y_ref).max()
    assert err <= TOL[precision], f"normwise {err:.3e}"


@pytest.mark.parametrize("precision", ["bf16", "bf16x3"])
@pytest.mark.parametrize("cfg", [(2, 64, 16, 16, 256, "scatter", "none"), (3, 32, 9, 16, 130, "raw", "max"),
                                 (2, 128, 32, 32, 128, "scatter", "avg"), (1, 16, 5, 32, 64, "raw", "none")],
                         ids=lambda c: "-".join(map(str, c)))
def test_tc_single_orientation_dyadic(O, dev, cfg, precision):
    """R = 1 (tiled_scatter_conv semantics) on the tensor cores, bit-exact on dyadic inputs."""
    import paper_2512_08888_b200 as P
    n, cin, h, w, cout, conv, pool = cfg
    d = O.Desc(n, cin, h, w, cout, 3, "single", 1, pool, 1, conv)
    rng = np.random.default_rng(abs(hash(cfg)) % 2**32)
    x = dyadic(rng, (n, cin, h, w))
    w0 = dyadic(rng, (cout, cin, 3, 3))
    bias = dyadic(rng, cout)
    y_ref, a_ref = O.ri_forward(d, x, w0, None, bias)
    y, a = run(P, d, x, w0, None, bias, precision, dev)
    assert np.array_equal(y.reshape(y_ref.shape), y_ref), f"max|dy| = {np.abs(y.reshape(y_ref.shape) - y_ref).max()}"
    if a_ref is not None:
        assert not a.any()


STRIP_CONFIGS = [
    # (n, cin, h, w, cout, group, R, pool, g, convention): W >= 48, W % 16 == 0 -> 4x16 strips
    (2, 64, 64, 64, 128, "p4m", 8, "subgroup", 4, "scatter"),
    (1, 32, 9, 48, 130, "p4", 4, "max", 4, "raw"),
    (2, 128, 16, 64, 128, "single", 1, "none", 1, "scatter"),
    (1, 16, 6, 80, 128, "steer", 8, "avg", 4, "scatter"),
]


@pytest.mark.parametrize("precision", ["bf16", "bf16x3"])
@pytest.mark.parametrize("cfg", STRIP_CONFIGS, ids=lambda c: "-".join(map(str, c)))
def test_tc_strip_dyadic_bitexact(O, dev, cfg, precision):
    import paper_2512_08888_b200 as P
    n, cin, h, w, cout, g, R, pool, pg, conv = cfg
    d = O.Desc(n, cin, h, w, cout, 3, g, R, pool, pg, conv)
    rng = np.random.default_rng(abs(hash(cfg)) % 2**32)
    x = dyadic(rng, (n, cin, h, w))
    w0 = dyadic(rng, (cout, cin, 3, 3))
    w1 = dyadic(rng, (cout, cin, 3, 3)) if g == "steer" else None
    bias = dyadic(rng, cout)
    y_ref, a_ref = O.ri_forward(d, x, w0, w1, bias)
    y, a = run(P, d, x, w0, w1, bias, precision, dev)
    if g == "steer":  # 45-degree base: irrational coefficients, FP32-class tolerance
        err = np.abs(y.reshape(y_ref.shape).astype(np.float64) - y_ref).max() / np.abs(y_ref).max()
        assert err <= TOL[precision], err
        return
    assert np.array_equal(y.reshape(y_ref.shape), y_ref), f"max|dy| = {np.abs(y.reshape(y_ref.shape) - y_ref).max()}"
    if a_ref is not None and g != "single":
        assert np.array_equal(a, a_ref), f"argmax mismatches {(a != a_ref).sum()}"


@pytest.mark.parametrize("precision", ["bf16", "bf16x3"])
@pytest.mark.parametrize("cfg", [(1, 512, 16, 16, 256, "single", 1, "none", 1),
                                 (1, 640, 8, 16, 128, "p4m", 8, "subgroup", 4),
                                 (1, 576, 6, 32, 130, "p4", 4, "max", 4),
                                 (1, 1024, 4, 64, 128, "single", 1, "none", 1)],
                         ids=lambda c: "-".join(map(str, c)))
def test_tc_large_cin_streamed_x(O, dev, cfg, precision):
    """Cin large enough that the X band does not fit in shared memory: X chunks are
    streamed with the weight stages (bf16x3) -- still bit-exact on dyadic inputs."""
    import paper_2512_08888_b200 as P
    n, cin, h, w, cout, g, R, pool, pg = cfg
    d = O.Desc(n, cin, h, w, cout, 3, g, R, pool, pg)
    rng = np.random.default_rng(abs(hash(cfg)) % 2**32)
    x = dyadic(rng, (n, cin, h, w))
    w0 = dyadic(rng, (cout, cin, 3, 3))
    bias = dyadic(rng, cout)
    y_ref, a_ref = O.ri_forward(d, x, w0, None, bias, nthreads=8)
    y, a = run(P, d, x, w0, None, bias, precision, dev)
    assert np.array_equal(y.reshape(y_ref.shape), y_ref), f"max|dy| = {np.abs(y.reshape(y_ref.shape) - y_ref).max()}"
    if a_ref is not None and g != "single":
        assert np.array_equal(a, a_ref)


SMALL_CONFIGS = [
    # (n, cin, s, cout, group, R, pool, g, convention): whole 8x8 / 4x4 images per band
    (32, 64, 8, 256, "single", 1, "none", 1, "scatter"),      # C1 shape
    (3, 16, 8, 130, "p4m", 8, "subgroup", 4, "raw"),
    (5, 32, 4, 256, "single", 1, "none", 1, "scatter"),       # ragged group of 4 images
    (6, 64, 4, 128, "p4", 4, "max", 4, "scatter"),
    (2, 100, 8, 128, "steer", 8, "avg", 4, "scatter"),
]


@pytest.mark.parametrize("precision", ["bf16", "bf16x3"])
@pytest.mark.parametrize("cfg", SMALL_CONFIGS, ids=lambda c: "-".join(map(str, c)))
def test_tc_small_images(O, dev, cfg, precision):
    import paper_2512_08888_b200 as P
    n, cin, sz, cout, g, R, pool, pg, conv = cfg
    d = O.Desc(n, cin, sz, sz, cout, 3, g, R, pool, pg, conv)
    rng = np.random.default_rng(abs(hash(cfg)) % 2**32)
    x = dyadic(rng, (n, cin, sz, sz))
    w0 = dyadic(rng, (cout, cin, 3, 3))
    w1 = dyadic(rng, (cout, cin, 3, 3)) if g == "steer" else None
    bias = dyadic(rng, cout)
    y_ref, a_ref = O.ri_forward(d, x, w0, w1, bias)
    y, a = run(P, d, x, w0, w1, bias, precision, dev)
    y = y.reshape(y_ref.shape)
    if g == "steer":
        err = np.abs(y.astype(np.float64) - y_ref).max() / np.abs(y_ref).max()
        assert err <= TOL[precision], err
        return
    assert np.array_equal(y, y_ref), f"max|dy| = {np.abs(y - y_ref).max()}"
    if a_ref is not None and g != "single":
        assert np.array_equal(a, a_ref), f"argmax mismatches {(a != a_ref).sum()}"


RELU_CASES = [
    # (kernel, pool, h, w): every tensor-core band geometry (w16, strip, img8, img4) and
    # every pooling branch of the fused epilogue, plus the CUDA-core kernel
    ("tc", "subgroup", 16, 16), ("tc", "avg", 16, 16), ("tc", "max", 16, 16), ("tc", "none", 16, 16),
    ("tc", "avg", 8, 48), ("tc", "subgroup", 8, 48), ("tc", "avg", 8, 8), ("tc", "avg", 4, 4),
    ("tc", "subgroup", 4, 4), ("simt", "subgroup", 16, 16), ("simt", "avg", 16, 16),
]


@pytest.mark.parametrize("case", RELU_CASES, ids=lambda c: "-".join(map(str, c)))
def test_fused_relu_activation(O, dev, case):
    """activation = relu is applied after the bias (relu of the oracle's pooled output)."""
    import paper_2512_08888_b200 as P
    kernel, pool, h, w = case
    n, cin, cout = 2, 64, 128
    rng = np.random.default_rng(5)
    x = dyadic(rng, (n, cin, h, w))
    w0 = dyadic(rng, (cout, cin, 3, 3))
    bias = dyadic(rng, cout)
    d = O.Desc(n, cin, h, w, cout, 3, "p4m", 8, pool, 4)
    y_ref, a_ref = O.ri_forward(d, x, w0, None, bias)
    t = lambda a: torch.from_numpy(a).to(dev)
    desc = P.Desc(n, cin, h, w, cout, 3, "p4m", 8, pool, 4, "scatter",
                  "bf16x3" if kernel == "tc" else "fp32", "relu")
    assert desc.kernel_name().startswith("tc_" if kernel == "tc" else "simt")
    bank = P.bank_precompute(desc, t(w0))
    y, a = P.ri_conv_forward(desc, t(x), bank, t(bias))
    assert np.array_equal(y.cpu().numpy().reshape(y_ref.shape), np.maximum(y_ref, 0))
    if a_ref is not None:
        assert np.array_equal(a.cpu().numpy().reshape(a_ref.shape), a_ref)


def test_tc_matches_simt_on_c3_shape_subset(O, dev):
    """C3 layer shape (256 -> 1024, steer R=8, subgroup-4) on 8 images: bf16x3 vs the
    FP32 CUDA-core kernel, normwise, plus determinism."""
    import paper_2512_08888_b200 as P
    g = torch.Generator(device=dev).manual_seed(3)
    n, cin, cout = 8, 256, 1024
    x = torch.rand((n, cin, 16, 16), generator=g, device=dev) * 2 - 1
    s = 1 / np.sqrt(cin * 9)
    fx = (torch.rand((cout, cin, 3, 3), generator=g, device=dev) * 2 - 1) * s
    fy = (torch.rand((cout, cin, 3, 3), generator=g, device=dev) * 2 - 1) * s
    outs = {}
    for prec in ("fp32", "bf16x3", "bf16x3"):
        d = P.Desc(n, cin, 16, 16, cout, 3, "steer", 8, "subgroup", 4, "scatter", prec)
        bank = P.bank_precompute(d, fx, fy)
        y, a = P.ri_conv_forward(d, x, bank)
        outs.setdefault(prec, []).append((y.clone(), a.clone()))
    y32 = outs["fp32"][0][0]
    y3 = outs["bf16x3"][0][0]
    assert torch.equal(outs["bf16x3"][0][0], outs["bf16x3"][1][0])
    err = ((y3 - y32).abs().max() / y32.abs().max()).item()
    assert err <= TOL["bf16x3"], err
