"""GPU parity: the FP32 CUDA-core kernels (precision="fp32") vs the CPU oracle (which is
pinned to the reference).  The shipped default (precision="auto", the tcgen05 kernels) is
checked at full config sizes in test_gpu_shipped_default.py.

Tolerances (FP32 path, stated here as the contract):
  * dyadic inputs (values k/4): bit-exact values AND argmax (every product and partial
    sum is exactly representable, so summation order cannot matter) -- for single, p4,
    p4m and steer N=4; steered bases at 2*pi*b/N (b >= 1) are irrational and fall back
    to the random-input tolerance;
  * random inputs: normwise max|dy| / max|y| <= 2e-6 and, where the oracle's top-2
    orientation gap exceeds 1e-4 * max|y|, argmax identical.
"""
import ctypes as C

import numpy as np
import pytest
import torch

from conftest import dyadic

pytestmark = pytest.mark.gpu

NORMWISE_TOL = 2e-6


def gpu_forward(P, d, x, w0, w1=None, bias=None, dev="cuda:0", precision="fp32"):
    t = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    desc = P.Desc(**{k: getattr(d, k) for k in ("n", "c_in", "h", "w", "c_out", "k", "group",
                                                  "orientations", "pool", "pool_group", "convention")},
                  precision=precision)
    bank = P.bank_precompute(desc, t(w0), t(w1))
    y, a = P.ri_conv_forward(desc, t(x), bank, t(bias))
    torch.cuda.synchronize()
    y = y.cpu().numpy()
    a = a.cpu().numpy() if a is not None else None
    if d.pool in ("avg", "max"):
        y = y[:, :, 0]
        a = a[:, :, 0] if a is not None else None
    return y, a, desc.kernel_name()


CONFIGS = [
    # (n, cin, h, w, cout, k, group, R, pool, g)
    (3, 5, 8, 8, 7, 3, "steer", 8, "subgroup", 4),
    (2, 16, 16, 16, 32, 3, "steer", 8, "subgroup", 4),
    (2, 17, 16, 16, 40, 3, "steer", 16, "subgroup", 4),
    (3, 8, 32, 32, 20, 3, "steer", 16, "subgroup", 8),
    (1, 6, 64, 64, 9, 3, "p4", 4, "max", 4),
    (5, 4, 4, 4, 33, 3, "p4m", 8, "max", 4),
    (2, 3, 5, 16, 6, 3, "p4m", 8, "avg", 4),
    (2, 3, 7, 8, 6, 3, "p4", 4, "none", 4),
    (2, 9, 9, 16, 5, 3, "steer", 12, "subgroup", 2),
    (3, 9, 8, 8, 12, 3, "steer", 8, "subgroup", 1),
    (4, 64, 8, 8, 256, 3, "single", 1, "none", 1),
    (2, 3, 6, 32, 4, 3, "single", 1, "max", 1),
    # generic kernel shapes
    (2, 3, 7, 5, 4, 5, "p4", 4, "max", 4),
    (2, 4, 6, 9, 3, 1, "p4m", 8, "subgroup", 4),
    (3, 2, 5, 6, 3, 2, "single", 1, "none", 1),
    (1, 3, 1, 9, 2, 3, "steer", 8, "avg", 4),
]


def _desc(O, cfg, convention="scatter"):
    n, cin, h, w, cout, k, g, R, pool, pg = cfg
    return O.Desc(n, cin, h, w, cout, k, g, R, pool, pg, convention)


@pytest.mark.parametrize("cfg", CONFIGS, ids=lambda c: "-".join(map(str, c)))
@pytest.mark.parametrize("convention", ["scatter", "raw"])
def test_dyadic_bitexact(O, dev, cfg, convention):
    import paper_2512_08888_b200 as P
    d = _desc(O, cfg, convention)
    rng = np.random.default_rng(hash(cfg) % 2**32)
    x = dyadic(rng, (d.n, d.c_in, d.h, d.w))
    w0, w1 = dyadic(rng, (d.c_out, d.c_in, d.k, d.k)), dyadic(rng, (d.c_out, d.c_in, d.k, d.k))
    bias = dyadic(rng, d.c_out)
    y_ref, a_ref = O.ri_forward(d, x, w0, w1, bias)
    y, a, kname = gpu_forward(P, d, x, w0, w1, bias)
    if d.group == "steer" and d.orientations > 4:
        # bases at theta = 2*pi*b/N, b >= 1, carry irrational sin/cos coefficients: the
        # operands are no longer dyadic, so only the FP32 tolerance applies
        err = np.abs(y.astype(np.float64) - y_ref).max() / np.abs(y_ref).max()
        assert err <= NORMWISE_TOL, f"{kname}: normwise {err:.3e}"
        return
    assert np.array_equal(y, y_ref), f"{kname}: max|dy|={np.abs(y - y_ref).max()}"
    if a_ref is not None:
        assert np.array_equal(a, a_ref), f"{kname}: argmax mismatches {(a != a_ref).sum()}"


def _top2_gap(f_unpooled, g):
    co, R = f_unpooled.shape[1], f_unpooled.shape[2]
    blk = np.sort(f_unpooled.reshape(f_unpooled.shape[0], co, R // g, g, *f_unpooled.shape[3:]), axis=3)
    return blk[:, :, :, -1] - blk[:, :, :, -2]


@pytest.mark.parametrize("cfg", CONFIGS[:10], ids=lambda c: "-".join(map(str, c)))
def test_random_fp32_tolerance(O, dev, cfg):
    import paper_2512_08888_b200 as P
    d = _desc(O, cfg)
    rng = np.random.default_rng(1 + hash(cfg) % 2**31)
    x = rng.uniform(-1, 1, (d.n, d.c_in, d.h, d.w)).astype(np.float32)
    s = 1 / np.sqrt(d.c_in * d.k * d.k)
    w0 = rng.uniform(-s, s, (d.c_out, d.c_in, d.k, d.k)).astype(np.float32)
    w1 = rng.uniform(-s, s, (d.c_out, d.c_in, d.k, d.k)).astype(np.float32)
    bias = rng.uniform(-0.1, 0.1, d.c_out).astype(np.float32)
    y_ref, a_ref = O.ri_forward(d, x, w0, w1, bias)
    y, a, kname = gpu_forward(P, d, x, w0, w1, bias)
    err = np.abs(y.astype(np.float64) - y_ref).max() / max(np.abs(y_ref).max(), 1e-30)
    assert err <= NORMWISE_TOL, f"{kname}: normwise {err:.3e}"
    if a_ref is not None:
        dn = O.Desc(d.n, d.c_in, d.h, d.w, d.c_out, d.k, d.group, d.orientations, "none")
        f, _ = O.ri_forward(dn, x, w0, w1)
        g = d.orientations if d.pool == "max" else d.pool_group
        if g > 1:
            gap = _top2_gap(f, g)
            if d.pool == "max":
                gap = gap[:, :, 0]
            safe = gap > 1e-4 * np.abs(y_ref).max()
            assert np.array_equal(a[safe], a_ref[safe]), f"{kname}: argmax"
            assert safe.mean() > 0.9


def test_bank_precompute_bitexact(O, dev):
    import paper_2512_08888_b200 as P
    rng = np.random.default_rng(3)
    for g, R in (("steer", 8), ("steer", 16), ("steer", 12), ("p4m", 8), ("p4", 4), ("single", 1)):
        fx = rng.standard_normal((6, 5, 3, 3)).astype(np.float32)
        fy = rng.standard_normal((6, 5, 3, 3)).astype(np.float32)
        od = O.Desc(1, 5, 4, 4, 6, 3, g, R)
        ref = O.build_bases(od, fx, fy)
        d = P.Desc(1, 5, 4, 4, 6, 3, g, R)
        bank = P.bank_precompute(d, torch.from_numpy(fx).to(dev), torch.from_numpy(fy).to(dev))
        assert np.array_equal(P.bank_bases(d, bank).cpu().numpy(), ref), g
        full = P.rotconv.build_orientation_bank_from(d, torch.from_numpy(fx).to(dev),
                                                     torch.from_numpy(fy).to(dev)).cpu().numpy()
        assert np.array_equal(full, O.build_orientation_bank(od, fx, fy)), g


@pytest.mark.parametrize("pool,g", [("avg", 1), ("max", 1), ("subgroup", 4), ("subgroup", 2)])
def test_standalone_pools(O, dev, pool, g):
    import paper_2512_08888_b200 as P
    rng = np.random.default_rng(4)
    f = rng.standard_normal((3, 5, 8, 6, 7)).astype(np.float32)
    f[:, :, 1] = f[:, :, 0]  # ties -> smallest index
    ft = torch.from_numpy(f).to(dev)
    for i in range(3):
        if pool == "avg":
            assert np.array_equal(P.orientation_pool_avg(ft[i]).cpu().numpy(), O.orientation_pool_avg(f[i]))
        elif pool == "max":
            y, a = P.orientation_pool_max(ft[i])
            yr, ar = O.orientation_pool_max(f[i])
            assert np.array_equal(y.cpu().numpy(), yr) and np.array_equal(a.cpu().numpy(), ar)
        else:
            y, a = P.subgroup_pool_max(ft[i], g)
            yr, ar = O.subgroup_pool_max(f[i], g)
            assert np.array_equal(y.cpu().numpy(), yr) and np.array_equal(a.cpu().numpy(), ar)


def test_golden_fixtures_on_gpu(O, dev, golden):
    import paper_2512_08888_b200 as P
    for i in range(7):
        x, w = golden[f"tiled_{i}_x"], golden[f"tiled_{i}_w"]
        xt, wt = torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)
        cnt = P.MultCounter()
        k = w.shape[2]
        y = P.tiled_scatter_conv(xt, wt, P.TileConfig(32, 32, k // 2), 4, cnt, precision="fp32").cpu().numpy()
        ref = golden[f"tiled_{i}_y"]
        assert np.abs(y - ref).max() <= NORMWISE_TOL * max(np.abs(ref).max(), 1e-30)
        assert [cnt.scalar_multiplications, cnt.scalar_additions] == list(golden[f"tiled_{i}_counts"])
        yr = P.scatter_conv_raw_multi(xt, wt, precision="fp32").cpu().numpy()
        refr = golden[f"raw_{i}_y"]
        assert np.abs(yr - refr).max() <= NORMWISE_TOL * max(np.abs(refr).max(), 1e-30)
    for i in range(5):
        key = f"slices_{i}_dyadic"
        gi, R, cin, h, w, cout = golden[key + "_meta"]
        g = list(O.GROUPS)[gi]
        d = O.Desc(1, int(cin), int(h), int(w), int(cout), 3, g, int(R))
        y, _, _ = gpu_forward(P, d, golden[key + "_x"][None], golden[key + "_w0"], golden[key + "_w1"])
        ref = golden[key + "_f"]
        if g == "steer" and R > 4:  # irrational steering coefficients: FP32 tolerance
            assert np.abs(y[0] - ref).max() <= NORMWISE_TOL * np.abs(ref).max(), key
        else:
            assert np.array_equal(y[0], ref), key


def test_host_entry_point_matches_device_path(O, dev):
    """rc_ri_conv_forward_host (the e2e drop-in) == device path == oracle (dyadic)."""
    from paper_2512_08888_b200 import _lib
    rng = np.random.default_rng(5)
    d = O.Desc(3, 8, 16, 16, 24, 3, "p4m", 8, "subgroup", 4)
    x = dyadic(rng, (3, 8, 16, 16))
    fx, fy, b = dyadic(rng, (24, 8, 3, 3)), dyadic(rng, (24, 8, 3, 3)), dyadic(rng, 24)
    y = np.zeros((3, 24, 2, 16, 16), np.float32)
    a = np.zeros((3, 24, 2, 16, 16), np.uint8)
    cd = _lib.rc_desc(3, 8, 16, 16, 24, 3, 2, 8, 3, 4, 0, 1)
    p = lambda arr: C.c_void_p(arr.ctypes.data)
    _lib.check(_lib.lib().rc_ri_conv_forward_host(C.byref(cd), p(x), p(fx), p(fy), p(b), p(y), p(a), 0))
    yr, ar = O.ri_forward(d, x, fx, fy, b)
    assert np.array_equal(y, yr) and np.array_equal(a, ar)


def test_tiled_scatter_conv_dropin_vs_reference(O, dev):
    """The shipped entry point (R=1) against the real reference build, with counters."""
    import paper_2512_08888_b200 as P
    if not O.ref_available():
        pytest.skip("no _ref")
    rng = np.random.default_rng(6)
    for (cin, h, w, cout) in [(64, 8, 8, 256), (7, 11, 13, 5), (16, 16, 16, 64)]:
        x = dyadic(rng, (cin, h, w))
        wt = dyadic(rng, (cout, cin, 3, 3))
        yr, m, a, _ = O.ref_tiled_scatter_conv(x, wt, workers=2)
        cnt, aux = P.MultCounter(), P.AuxMemCounter()
        y = P.tiled_scatter_conv(torch.from_numpy(x).to(dev), torch.from_numpy(wt).to(dev),
                                 P.TileConfig(), 2, cnt, aux).cpu().numpy()
        assert np.array_equal(y, yr)
        assert (cnt.scalar_multiplications, cnt.scalar_additions) == (m, a)
    with pytest.raises(ValueError, match="tiled_scatter_conv: invalid halo"):
        P.tiled_scatter_conv(torch.zeros(2, 4, 4, device=dev), torch.zeros(1, 2, 3, 3, device=dev),
                             P.TileConfig(32, 32, 2), 1)


def test_full_c3_subset_and_virtual_shards(O, dev):
    """FP32 CUDA-core kernel: C3 at full size (N=256, 16x16x256->1024, steer R=8, subgroup-4): images 0 and 255
    against the oracle; the whole batch equals the concatenation of two half-batch
    launches (virtual shards, bit-identical); run-to-run determinism."""
    import paper_2512_08888_b200 as P
    g = torch.Generator(device=dev).manual_seed(0)
    n, cin, h, w, cout = 256, 256, 16, 16, 1024
    x = torch.rand((n, cin, h, w), generator=g, device=dev) * 2 - 1
    s = 1 / np.sqrt(cin * 9)
    fx = (torch.rand((cout, cin, 3, 3), generator=g, device=dev) * 2 - 1) * s
    fy = (torch.rand((cout, cin, 3, 3), generator=g, device=dev) * 2 - 1) * s
    bias = (torch.rand(cout, generator=g, device=dev) * 0.2 - 0.1)
    d = P.Desc(n, cin, h, w, cout, 3, "steer", 8, "subgroup", 4, "scatter", "fp32")
    bank = P.bank_precompute(d, fx, fy)
    y, a = P.ri_conv_forward(d, x, bank, bias)
    y2, a2 = P.ri_conv_forward(d, x, bank, bias)
    assert torch.equal(y, y2) and torch.equal(a, a2)
    dh = P.Desc(n // 2, cin, h, w, cout, 3, "steer", 8, "subgroup", 4, "scatter", "fp32")
    yh0, ah0 = P.ri_conv_forward(dh, x[: n // 2].contiguous(), bank, bias)
    yh1, ah1 = P.ri_conv_forward(dh, x[n // 2:].contiguous(), bank, bias)
    assert torch.equal(torch.cat([yh0, yh1]), y) and torch.equal(torch.cat([ah0, ah1]), a)
    xs, fxs, fys, bs = x.cpu().numpy(), fx.cpu().numpy(), fy.cpu().numpy(), bias.cpu().numpy()
    od = O.Desc(n, cin, h, w, cout, 3, "steer", 8, "subgroup", 4)
    for img in (0, n - 1):
        yr, ar = O.ri_forward(od, xs, fxs, fys, bs, nthreads=8, images=(img, img + 1))
        yi = y[img].cpu().numpy()
        err = np.abs(yi.astype(np.float64) - yr[img]).max() / np.abs(yr[img]).max()
        assert err <= NORMWISE_TOL
        agree = (a[img].cpu().numpy() == ar[img]).mean()
        assert agree > 0.999
