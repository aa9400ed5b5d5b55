"""Carry-band tensor-core kernels (ri_tc.cu, round 2): bands without halo rows whose boundary
rows are carried across bands in TMEM, for 16-wide images and 16-column strips of wider ones.

The carry logic depends on the band index (first band: no carry-in; last band: the carried
row completes from registers) and on the base loop (bases outermost: every base restarts the
carry), so these cases sweep H across the band boundaries (H = 1 .. 4k+1), bases 1..4,
partial channel tiles, every pooling mode (avg spanning the bases, max spanning the bases,
subgroup, none) with bias and ReLU.  Dyadic inputs: bit-exact in values and argmax, both
precisions (the [Xh | Xl] concatenated MMAs included)."""
import numpy as np
import pytest
import torch

from conftest import dyadic

pytestmark = pytest.mark.gpu

# dyadic-exact groups: p4, p4m (2 bases), steer R=4 (one base at theta = 0); steerable banks
# with more bases have irrational coefficients (covered by the tolerance cases below)
CASES = [
    # (n, cin, h, w, cout, group, R, pool, g, activation)
    (2, 32, 1, 16, 128, "p4m", 8, "subgroup", 4, "none"),
    (2, 32, 3, 16, 200, "p4m", 8, "subgroup", 4, "relu"),
    (1, 64, 4, 16, 128, "p4m", 8, "max", 8, "none"),
    (2, 32, 5, 16, 130, "p4m", 8, "max", 8, "none"),
    (1, 16, 7, 16, 128, "p4", 4, "avg", 4, "relu"),
    (2, 48, 8, 16, 256, "p4m", 8, "avg", 8, "none"),
    (1, 32, 17, 16, 128, "p4m", 8, "none", 8, "none"),
    (1, 16, 33, 16, 128, "steer", 4, "subgroup", 2, "relu"),
    (1, 32, 1, 32, 128, "p4m", 8, "subgroup", 4, "none"),
    (2, 16, 3, 48, 130, "p4m", 8, "max", 8, "relu"),
    (1, 64, 5, 96, 128, "p4", 4, "avg", 4, "none"),
    (1, 32, 9, 32, 256, "p4m", 8, "none", 4, "none"),
]


@pytest.mark.parametrize("precision", ["bf16x3", "bf16"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(map(str, c)))
def test_carry_bands_dyadic_bitexact(O, dev, case, precision):
    import paper_2512_08888_b200 as P
    n, cin, h, w, cout, g, R, pool, pg, act = case
    desc = P.Desc(n, cin, h, w, cout, 3, g, R, pool, pg, "scatter", precision, act)
    assert desc.kernel_name() == ("tc_k3w16_" if w == 16 else "tc_k3strip_") + precision, desc.kernel_name()
    rng = np.random.default_rng(abs(hash(case)) % 2**32)
    x = dyadic(rng, (n, cin, h, w))
    w0 = dyadic(rng, (cout, cin, 3, 3))
    w1 = dyadic(rng, (cout, cin, 3, 3)) if g == "steer" else None
    bias = dyadic(rng, cout)
    od = O.Desc(n, cin, h, w, cout, 3, g, R, pool, pg)
    y_ref, a_ref = O.ri_forward(od, x, w0, w1, bias)
    if act == "relu":
        y_ref = np.maximum(y_ref, 0)
    t = lambda a: torch.from_numpy(a).to(dev)
    bank = P.bank_precompute(desc, t(w0), t(w1) if w1 is not None else None)
    y, a = P.ri_conv_forward(desc, t(x), bank, t(bias))
    torch.cuda.synchronize()
    y = y.cpu().numpy().reshape(y_ref.shape)
    assert np.array_equal(y, y_ref), f"max|dy| = {np.abs(y - y_ref).max()}"
    if a_ref is not None:
        assert np.array_equal(a.cpu().numpy().reshape(a_ref.shape), a_ref)


TOL_CASES = [
    # four bases (steer R=16): every base restarts the carried rows
    (2, 32, 5, 16, 200, "steer", 16, "subgroup", 4),
    (1, 32, 9, 16, 128, "steer", 16, "max", 16),
    (1, 16, 6, 32, 128, "steer", 16, "avg", 16),
    (2, 32, 3, 48, 130, "steer", 12, "subgroup", 4),
]


@pytest.mark.parametrize("precision,tol", [("bf16x3", 3e-5), ("bf16", 1e-2)])
@pytest.mark.parametrize("case", TOL_CASES, ids=lambda c: "-".join(map(str, c)))
def test_carry_bands_many_bases_tolerance(O, dev, case, precision, tol):
    import paper_2512_08888_b200 as P
    n, cin, h, w, cout, g, R, pool, pg = case
    desc = P.Desc(n, cin, h, w, cout, 3, g, R, pool, pg, "scatter", precision)
    rng = np.random.default_rng(11 + abs(hash(case)) % 2**31)
    x = rng.uniform(-1, 1, (n, cin, h, w)).astype(np.float32)
    s = 1 / np.sqrt(cin * 9)
    w0 = rng.uniform(-s, s, (cout, cin, 3, 3)).astype(np.float32)
    w1 = rng.uniform(-s, s, (cout, cin, 3, 3)).astype(np.float32)
    bias = rng.uniform(-0.1, 0.1, cout).astype(np.float32)
    y_ref, _ = O.ri_forward(O.Desc(n, cin, h, w, cout, 3, g, R, pool, pg), x, w0, w1, bias)
    t = lambda a: torch.from_numpy(a).to(dev)
    y, _ = P.ri_conv_forward(desc, t(x), P.bank_precompute(desc, t(w0), t(w1)), t(bias))
    y = y.cpu().numpy().reshape(y_ref.shape).astype(np.float64)
    assert np.abs(y - y_ref).max() / np.abs(y_ref).max() <= tol
