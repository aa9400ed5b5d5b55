"""SPEC known-answer examples and properties on the CPU oracle."""
import math

import numpy as np
import pytest

from conftest import dyadic

A9 = np.arange(1, 10, dtype=np.float64).reshape(3, 3)


def test_rot90_kats(O):
    assert O.rot90_plane(A9, 1).tolist() == [[3, 6, 9], [2, 5, 8], [1, 4, 7]]
    assert np.array_equal(O.rot90_plane(A9, 0), A9)
    assert O.rot90_plane(np.array([[1., 2.], [3., 4.]]), 2).tolist() == [[4, 3], [2, 1]]
    g = np.random.default_rng(0).standard_normal((3, 5))
    r = g
    for _ in range(4):
        r = O.rot90_plane(r, 1)
    assert np.array_equal(r, g)
    assert O.rot90_plane(g, 1).shape == (5, 3)


def test_mirror_kats(O):
    assert O.mirror_plane(np.array([[1., 2., 3.]])).tolist() == [[3, 2, 1]]
    assert O.mirror_plane(np.array([[1., 2., 1.]])).tolist() == [[1, 2, 1]]
    g = np.random.default_rng(1).standard_normal((4, 4))
    assert np.array_equal(O.mirror_plane(O.mirror_plane(g)), g)


def test_pack_roundtrip_vs_reference(O):
    """CNHW/NHWC packing = exact permutations."""
    if not O.ref_available():
        pytest.skip("no _ref")
    import ctypes as C
    rng = np.random.default_rng(2)
    b = rng.standard_normal((3, 4, 5, 6)).astype(np.float32)
    out = np.empty((4, 3 * 5 * 6), np.float32)
    O.ref().ref_pack_cnhw_f(O._p(b), 3, 4, 5, 6, O._p(out))
    assert np.array_equal(out, b.transpose(1, 0, 2, 3).reshape(4, -1))
    w = rng.standard_normal((5, 4, 3, 3)).astype(np.float32)
    out2 = np.empty((5, 36), np.float32)
    O.ref().ref_pack_nhwc_f(O._p(w), 5, 4, 3, 3, O._p(out2))
    assert np.array_equal(out2, w.transpose(0, 2, 3, 1).reshape(5, -1))
    del C


def test_gather_same_kats(O):
    x = A9.reshape(1, 3, 3)
    delta = np.zeros((1, 1, 3, 3)); delta[0, 0, 1, 1] = 1
    assert np.array_equal(O.conv_gather_same(x, delta), x)
    assert O.conv_gather_same(x, np.ones((1, 1, 3, 3)))[0, 0, 0] == 12


def test_scatter_single_kats(O):
    y, m, a = O.scatter_conv_single(A9, np.ones((3, 3)))
    assert y[1, 1] == 45 and y[0, 0] == 12 and m == 81 and a == 49
    delta = np.zeros((3, 3)); delta[1, 1] = 1
    g = np.random.default_rng(3).standard_normal((5, 4))
    assert np.array_equal(O.scatter_conv_single(g, delta)[0], g)


def test_scatter_multi_kats(O):
    rng = np.random.default_rng(4)
    x1 = rng.standard_normal((1, 5, 5))
    w1 = rng.standard_normal((2, 1, 3, 3))
    x2 = np.concatenate([x1, np.zeros_like(x1)])                               # SPEC:207 zero channel
    w2 = np.concatenate([w1, rng.standard_normal((2, 1, 3, 3))], axis=1)
    assert np.array_equal(O.scatter_conv_multi(x2, w2), O.scatter_conv_multi(x1, w1))
    wneg = np.concatenate([w1[:1], -w1[:1]])                                    # SPEC:209 negation
    y = O.scatter_conv_multi(x1, wneg)
    assert np.array_equal(y[1], -y[0])


def test_clipped_writes(O):
    assert O.clipped_writes(16, 16, 3, 3) == 2116
    assert O.clipped_writes(32, 32, 3, 3) == 8836
    assert O.clipped_writes(8, 8, 3, 3) == 484


def test_transform_kernel_kats(O):
    w = A9.reshape(1, 1, 3, 3)
    assert O.transform_kernel(w, 1)[0, 0].tolist() == [[3, 6, 9], [2, 5, 8], [1, 4, 7]]
    assert np.array_equal(O.transform_kernel(O.transform_kernel(w, 2), 2), w)
    g = np.random.default_rng(5).standard_normal((1, 1, 3, 3))
    ts = [O.transform_kernel(g, r, m) for m in (False, True) for r in range(4)]
    for i in range(8):
        for j in range(i + 1, 8):
            assert not np.array_equal(ts[i], ts[j])


def test_group_conv_kats(O):
    rng = np.random.default_rng(6)
    x = rng.standard_normal((2, 6, 6))
    ones = np.ones((1, 2, 3, 3))
    d = O.Desc(1, 2, 6, 6, 1, 3, "p4", 4)
    f = O.group_conv_scatter_reuse(d, x, O.build_bases(d, ones))
    for r in range(1, 4):
        assert np.allclose(f[:, r], f[:, 0], atol=1e-12)
    delta = np.zeros((1, 1, 3, 3)); delta[0, 0, 1, 1] = 1
    d1 = O.Desc(1, 1, 6, 6, 1, 3, "p4", 4)
    f = O.group_conv_scatter_reuse(d1, x[:1], O.build_bases(d1, delta))
    for r in range(4):
        assert np.array_equal(f[0, r], x[0])
    # slice r == conv_gather_same(X, transform(reverse W, r)) (P1)
    w = rng.standard_normal((3, 2, 3, 3))
    d2 = O.Desc(1, 2, 6, 6, 3, 3, "p4", 4)
    f = O.group_conv_scatter_reuse(d2, x, O.build_bases(d2, w))
    rev = w[:, :, ::-1, ::-1].copy()
    for r in range(4):
        g = O.conv_gather_same(x, O.transform_kernel(rev, r))
        assert np.allclose(f[:, r], g, rtol=0, atol=1e-12)


def test_group_reuse_equals_gather_50_p4_and_p4m(O):
    """SPEC:280-282, acceptance 3: reuse == per-slice gather (after the duality)."""
    rng = np.random.default_rng(7)
    for i in range(50):
        g = "p4" if i % 5 else "p4m"
        R = 4 if g == "p4" else 8
        c, co, h, w = rng.integers(1, 5), rng.integers(1, 4), rng.integers(1, 10), rng.integers(1, 10)
        x = rng.standard_normal((c, h, w))
        wt = rng.standard_normal((co, c, 3, 3))
        d = O.Desc(1, int(c), int(h), int(w), int(co), 3, g, R)
        f = O.group_conv_scatter_reuse(d, x, O.build_bases(d, wt))
        rev = wt[:, :, ::-1, ::-1].copy()
        for o in range(R):
            gk = O.transform_kernel(rev, o % 4, mirror=False) if o < 4 else \
                O.transform_kernel(O.transform_kernel(wt, 0, True)[:, :, ::-1, ::-1].copy(), o % 4)
            gg = O.conv_gather_same(x, gk)
            assert np.max(np.abs(f[:, o] - gg)) <= 1e-12 * max(1, np.max(np.abs(gg)))


def test_pool_kats(O):
    f = np.array([1., 2., 3., 4.]).reshape(1, 4, 1, 1)
    assert O.orientation_pool_avg(f)[0, 0, 0] == 2.5
    y, a = O.orientation_pool_max(f)
    assert y[0, 0, 0] == 4 and a[0, 0, 0] == 3
    y, a = O.orientation_pool_max(np.full((1, 4, 1, 1), 7.0))
    assert y[0, 0, 0] == 7 and a[0, 0, 0] == 0                                      # SPEC:299 tie
    f8 = np.random.default_rng(8).standard_normal((2, 8, 3, 3))
    y, a = O.subgroup_pool_max(f8, 4)
    assert y.shape == (2, 2, 3, 3)
    yf, af = O.orientation_pool_max(f8)
    ys, as_ = O.subgroup_pool_max(f8, 8)
    assert np.array_equal(yf, ys[:, 0]) and np.array_equal(af, as_[:, 0])
    blk = f8.reshape(2, 2, 4, 3, 3)
    assert np.array_equal(y, blk.max(axis=2)) and np.array_equal(a, blk.argmax(axis=2))


def test_steer_kats(O):
    rng = np.random.default_rng(9)
    fx, fy = rng.standard_normal(9), rng.standard_normal(9)
    assert np.array_equal(O.steer(fx, fy, 0.0), fy)
    assert np.allclose(O.steer(fx, fy, math.pi / 2), fx, atol=1e-15)
    assert np.allclose(O.steer(fx, fy, math.pi / 4), (fx + fy) / math.sqrt(2), atol=1e-15)


def gaussian_derivative_basis(k, sigma):
    """SPEC:484-492 test fixture: f_x ~ -x exp(.), f_y ~ -y exp(.), unit L2 (x = column)."""
    c = k // 2
    yy, xx = np.mgrid[0:k, 0:k].astype(np.float64)
    xx -= c
    yy -= c  # grid centred at (K/2, K/2), y = row index: then R1(f_x) = -f_y, R1(f_y) = f_x
    g = np.exp(-(xx ** 2 + yy ** 2) / (2 * sigma ** 2))
    fx, fy = -xx * g, -yy * g
    return fx / np.linalg.norm(fx), fy / np.linalg.norm(fy)


def test_orientation_bank_kats(O):
    fx, fy = gaussian_derivative_basis(5, 1.2)
    fx4, fy4 = fx.reshape(1, 1, 5, 5), fy.reshape(1, 1, 5, 5)
    d4 = O.Desc(1, 1, 1, 1, 1, 5, "steer", 4)
    bank = O.build_orientation_bank(d4, fx4, fy4)
    for r in range(4):                                                             # SPEC:454 p4 orbit of f_y
        assert np.array_equal(bank[r], O.transform_kernel(fy4, r))
    d8 = O.Desc(1, 1, 1, 1, 1, 5, "steer", 8)
    assert O.build_bases(d8, fx4, fy4).shape[0] == 2
    assert O.build_orientation_bank(d8, fx4, fy4).shape[0] == 8
    d16 = O.Desc(1, 1, 1, 1, 1, 5, "steer", 16)
    b16 = O.build_orientation_bank(d16, fx4, fy4)
    # 135 deg = base 45 deg (b=2) rotated once: orbit-major o = b*4 + r
    assert np.array_equal(b16[2 * 4 + 1], O.transform_kernel(b16[2 * 4 + 0], 1))
    # covariant basis: quadrant reuse == direct steering (acceptance 7)
    for b in range(4):
        for r in range(4):
            theta = 2 * math.pi * b / 16 + r * math.pi / 2
            direct = O.steer(fx4, fy4, theta)
            assert np.max(np.abs(b16[b * 4 + r] - direct)) < 1e-12


@pytest.mark.parametrize("group,R", [("p4", 4), ("steer", 8)])
def test_equivariance(O, group, R):
    """SPEC:314-315, acceptance 5: avg pool exactly equivariant (dyadic, exact in FP64);
    orientation permutation law slice r(rot X) == rot(slice (r-1) of X) for p4."""
    rng = np.random.default_rng(10)
    c, co, s = 3, 2, 7
    x = dyadic(rng, (1, c, s, s)).astype(np.float64)
    fx, fy = dyadic(rng, (co, c, 3, 3)).astype(np.float64), dyadic(rng, (co, c, 3, 3)).astype(np.float64)
    xr = np.rot90(x, 1, axes=(2, 3)).copy()
    d = O.Desc(1, c, s, s, co, 3, group, R, "avg")
    ya, _ = O.ri_forward(d, x, fx, fy)
    yb, _ = O.ri_forward(d, xr, fx, fy)
    if group == "p4":
        assert np.array_equal(yb[0], np.rot90(ya[0], 1, axes=(1, 2)))
        dn = O.Desc(1, c, s, s, co, 3, "p4", 4, "none")
        fa, _ = O.ri_forward(dn, x, fx)
        fb, _ = O.ri_forward(dn, xr, fx)
        for r in range(4):
            assert np.array_equal(fb[0, :, r], np.rot90(fa[0, :, (r - 1) % 4], 1, axes=(1, 2)))


def test_validation_messages(O):
    assert O.validate(O.Desc(1, 1, 1, 1, 1, 2, "p4", 4)) == \
        "transform_kernel: rotation groups need odd square kernels"
    assert O.validate(O.Desc(1, 1, 1, 1, 1, 3, "steer", 6)) == \
        "build_orientation_bank: N must be a multiple of 4"
    assert O.validate(O.Desc(1, 1, 1, 1, 1, 3, "p4m", 8, "subgroup", 3)) == \
        "subgroup_pool_max: R not divisible by group_size"
    assert O.validate(O.Desc(1, 1, 1, 1, 1, 3, "p4m", 8, "subgroup", 4)) is None
