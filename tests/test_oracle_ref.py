"""Pin the C oracle to the UNMODIFIED reference (oracle/_ref) and to the committed
golden fixtures made from it.  CPU only."""
import numpy as np
import pytest

from conftest import dyadic


def _need_ref(O):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_scatter_multi_bitexact_vs_reference(O, dt, k):
    _need_ref(O)
    rng = np.random.default_rng(k)
    for _ in range(3):
        c, h, w, co = rng.integers(1, 6), rng.integers(1, 12), rng.integers(1, 12), rng.integers(1, 5)
        x = rng.standard_normal((c, h, w)).astype(dt)
        wt = rng.standard_normal((co, c, k, k)).astype(dt)
        y_ref, m = O.ref_scatter_conv_multi(x, wt)
        assert np.array_equal(O.scatter_conv_multi(x, wt), y_ref)
        assert np.array_equal(O.scatter_conv_raw_multi(x, wt), O.ref_scatter_conv_raw_multi(x, wt))
        assert m == h * w * k * k * c * co


@pytest.mark.parametrize("workers,tile,strategy", [(1, (32, 32), 0), (4, (5, 5), 0), (3, (1, 1), 0),
                                                   (2, (32, 32), 1), (8, (7, 3), 1)])
def test_tiled_matches_untiled_reference(O, workers, tile, strategy):
    """SPEC:216-218, 652 (acceptance 9): tiled == untiled for any tile/worker count."""
    _need_ref(O)
    rng = np.random.default_rng(9)
    x = rng.standard_normal((4, 16, 16))
    wt = rng.standard_normal((3, 4, 3, 3))
    y, m, a, _ = O.ref_tiled_scatter_conv(x, wt, tile=tile, workers=workers, strategy=strategy)
    assert np.array_equal(y, O.scatter_conv_multi(x, wt))
    assert m == 16 * 16 * 9 * 4 * 3 and a == O.clipped_writes(16, 16, 3, 3) * 3


def test_tiled_reference_validation_messages(O):
    _need_ref(O)
    x = np.zeros((2, 4, 4), np.float32)
    with pytest.raises(ValueError, match="tiled_scatter_conv: invalid halo"):
        O.ref_tiled_scatter_conv(x, np.zeros((1, 2, 3, 3), np.float32), halo=2)
    with pytest.raises(ValueError, match="tiled_scatter_conv: channel mismatch"):
        O.ref_tiled_scatter_conv(x, np.zeros((1, 3, 3, 3), np.float32))
    with pytest.raises(ValueError, match="tiled_scatter_conv: workers must be >= 1"):
        O.ref_tiled_scatter_conv(x, np.zeros((1, 2, 3, 3), np.float32), workers=0)


@pytest.mark.parametrize("group,R", [("single", 1), ("p4", 4), ("p4m", 8), ("steer", 4),
                                     ("steer", 8), ("steer", 16)])
@pytest.mark.parametrize("convention", ["scatter", "raw"])
def test_reuse_oracle_bitexact_vs_reference_slices(O, group, R, convention):
    """The oracle's true reuse loop (one dot per tap, scattered to 4 rotations) is
    bit-identical to R separate reference convolutions."""
    _need_ref(O)
    rng = np.random.default_rng(R * 7 + len(group))
    for dt in (np.float32, np.float64):
        cin, h, w, co = 5, 7, 6, 3
        d = O.Desc(1, cin, h, w, co, 3, group, R, convention=convention)
        x = rng.standard_normal((cin, h, w)).astype(dt)
        w0 = rng.standard_normal((co, cin, 3, 3)).astype(dt)
        w1 = rng.standard_normal((co, cin, 3, 3)).astype(dt)
        bases = O.build_bases(d, w0, w1)
        assert np.array_equal(O.group_conv_scatter_reuse(d, x, bases), O.ref_ri_slices(d, x, w0, bases))


def test_acceptance1_scatter_equals_gather_of_reversed(O):
    """SPEC:644 acceptance 1: >=100 random cases, sizes 1-32, C<=8, K in {1,3,5}, <1e-12."""
    _need_ref(O)
    rng = np.random.default_rng(644)
    for i in range(100):
        k = (1, 3, 5)[i % 3]
        c, co = rng.integers(1, 9), rng.integers(1, 9)
        h, w = rng.integers(1, 33), rng.integers(1, 33)
        x = rng.standard_normal((c, h, w))
        wt = rng.standard_normal((co, c, k, k))
        rev = wt[:, :, ::-1, ::-1].copy()
        y = O.scatter_conv_multi(x, wt)
        g = O.ref_conv_gather_same(x, rev)
        assert np.max(np.abs(y - g)) <= 1e-12 * max(1.0, np.max(np.abs(g)))


def test_golden_fixtures_tiled(O, golden):
    for i in range(7):
        x, w = golden[f"tiled_{i}_x"], golden[f"tiled_{i}_w"]
        assert np.array_equal(O.scatter_conv_multi(x, w), golden[f"tiled_{i}_y"])
        assert np.array_equal(O.scatter_conv_raw_multi(x, w), golden[f"raw_{i}_y"])
        m, a = golden[f"tiled_{i}_counts"]
        c, h, ww = x.shape
        co, _, k, _ = w.shape
        assert m == h * ww * k * k * c * co and a == O.clipped_writes(h, ww, k, k) * co


def test_golden_fixtures_slices(O, golden):
    for i in range(5):
        for kind in ("rand", "dyadic"):
            key = f"slices_{i}_{kind}"
            gi, R, cin, h, w, cout = golden[key + "_meta"]
            d = O.Desc(1, int(cin), int(h), int(w), int(cout), 3, list(O.GROUPS)[gi], int(R))
            bases = O.build_bases(d, golden[key + "_w0"], golden[key + "_w1"])
            assert np.array_equal(bases, golden[key + "_bases"])
            f = O.group_conv_scatter_reuse(d, golden[key + "_x"], bases)
            assert np.array_equal(f, golden[key + "_f"]), key


def test_batch_forward_threads_invariant(O):
    rng = np.random.default_rng(5)
    d = O.Desc(5, 4, 8, 8, 6, 3, "steer", 8, "subgroup", 4)
    x, fx, fy = dyadic(rng, (5, 4, 8, 8)), dyadic(rng, (6, 4, 3, 3)), dyadic(rng, (6, 4, 3, 3))
    y1, a1 = O.ri_forward(d, x, fx, fy, nthreads=1)
    y4, a4 = O.ri_forward(d, x, fx, fy, nthreads=4)
    assert np.array_equal(y1, y4) and np.array_equal(a1, a4)


@pytest.mark.parametrize("group,R,pool,g", [("p4", 4, "max", 4), ("p4m", 8, "subgroup", 4), ("steer", 8, "subgroup", 4),
                                            ("steer", 16, "subgroup", 8), ("p4m", 8, "avg", 4), ("p4", 4, "none", 4),
                                            ("single", 1, "none", 1)])
def test_reference_built_layer_equals_oracle_layer(O, group, R, pool, g):
    """bench.py's reference arm: the layer built from the reference's own code path (R x
    tiled_scatter_conv per image, ref_ri_batch) equals the oracle's fused reuse layer
    (ri_forward) bit-for-bit -- values, argmax, bias -- over a multi-image batch."""
    _need_ref(O)
    rng = np.random.default_rng(R + len(pool))
    n, cin, h, w, co = 3, 5, 7, 6, 4
    d = O.Desc(n, cin, h, w, co, 3, group, R, pool, g)
    x = rng.standard_normal((n, cin, h, w)).astype(np.float32)
    w0 = rng.standard_normal((co, cin, 3, 3)).astype(np.float32)
    w1 = rng.standard_normal((co, cin, 3, 3)).astype(np.float32)
    b = rng.standard_normal(co).astype(np.float32)
    y_ref, a_ref = O.ref_ri_batch(d, x, w0, w1, b, nthreads=2)
    y, a = O.ri_forward(d, x, w0, w1, b)
    assert np.array_equal(y_ref, y), np.abs(y_ref - y).max()
    if a is not None:
        assert np.array_equal(a_ref, a)
