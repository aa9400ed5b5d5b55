"""SPEC's finite-difference verifier (acceptance 6 at SPEC:649).

CPU: the verifier itself against SPEC's example (quadratic, error < 1e-9) and a linear map.
GPU: the library's backward (rc_ri_conv_backward: pool / ReLU / bias backward, input and
weight gradients) against central differences of the float64 CPU oracle's forward of the
same layer (oracle/rco_ri_forward_f64) -- the oracle, not the library, is differentiated.
The library computes in 32-bit arithmetic, so its tolerance is SPEC's 32-bit one: worst
relative error <= 1e-5 (fp32 CUDA-core path), <= 1e-4 (bf16x3 tensor-core path), over >= 50
sampled coordinates per gradient; max-pool ties and ReLU kinks are skipped.
"""
import math

import numpy as np
import pytest

import fd  # oracle/fd.py (test infrastructure)


def test_fd_quadratic_kat():
    rng = np.random.default_rng(0)
    x = rng.standard_normal(50)  # |f| ~ 50: round-off ~ 50 ulp / (2 eps |g|) < 1e-9
    err, used = fd.finite_diff_check(lambda v: float((v * v).sum()), x, 2 * x, 1e-5)
    assert used == 50 and err < 1e-9, err


def test_fd_linear_map_and_errors():
    rng = np.random.default_rng(1)
    a = rng.standard_normal((30, 40))
    m = rng.standard_normal(30)
    x = rng.standard_normal(40)
    err, _ = fd.finite_diff_check(lambda v: float(m @ (a @ v)), x, a.T @ m, 1e-5, samples=40)
    assert err < 1e-8
    bad = a.T @ m
    bad[5] = -bad[5]  # a wrong sign is caught: error = 2 |g_5| / |g_5|
    err, _ = fd.finite_diff_check(lambda v: float(m @ (a @ v)), x, bad, 1e-5, coords=[5])
    assert abs(err - 2.0) < 1e-6
    with pytest.raises(ValueError):
        fd.finite_diff_check(lambda v: 0.0, x, x, 0.0)


CASES = [
    # (n, cin, h, w, cout, group, R, pool, g, activation, precision, tol)
    (1, 4, 6, 6, 4, "p4", 4, "avg", 4, "none", "fp32", 1e-5),
    (1, 4, 6, 6, 4, "p4m", 8, "max", 8, "none", "fp32", 1e-5),
    (2, 3, 5, 7, 6, "steer", 8, "subgroup", 4, "relu", "fp32", 1e-5),
    (1, 5, 6, 6, 3, "single", 1, "none", 1, "none", "fp32", 1e-5),
    # tensor-core geometries (16-wide carry bands, whole 8x8 images, implicit GEMM)
    (1, 16, 5, 16, 8, "p4m", 8, "max", 8, "none", "bf16x3", 1e-4),
    (1, 16, 8, 8, 8, "steer", 8, "subgroup", 4, "relu", "bf16x3", 1e-4),
    (1, 16, 6, 16, 8, "p4", 4, "avg", 4, "none", "bf16x3", 1e-4),
    (1, 16, 5, 12, 8, "single", 1, "none", 1, "none", "bf16x3", 1e-4),
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(map(str, c[:11])))
def test_backward_vs_oracle_finite_differences(O, dev, case):
    import torch
    import paper_2512_08888_b200 as P
    n, cin, h, w, cout, g, R, pool, pg, act, precision, tol = case
    desc = P.Desc(n, cin, h, w, cout, 3, g, R, pool, pg, "scatter", precision, act)
    assert precision != "bf16x3" or desc.kernel_name().startswith("tc_"), desc.kernel_name()
    od = O.Desc(n, cin, h, w, cout, 3, g, R, pool, pg, "scatter")
    rng = np.random.default_rng(abs(hash(case)) % 2**31)
    x = rng.uniform(-1, 1, (n, cin, h, w)).astype(np.float32)
    s = 1 / math.sqrt(cin * 9)
    w0 = rng.uniform(-s, s, (cout, cin, 3, 3)).astype(np.float32)
    w1 = rng.uniform(-s, s, (cout, cin, 3, 3)).astype(np.float32) if g == "steer" else None
    bias = rng.uniform(-0.1, 0.1, cout).astype(np.float32)
    t = lambda a: torch.from_numpy(a).to(dev)
    bank = P.bank_precompute(desc, t(w0), t(w1) if w1 is not None else None)
    y, am = P.ri_conv_forward(desc, t(x), bank, t(bias))
    m = rng.uniform(-1, 1, tuple(y.shape))
    dx, dw0, dw1, db = P.ri_conv_backward(desc, t(x), bank, t(m.astype(np.float32)), y, am)
    torch.cuda.synchronize()
    grads = {"x": dx, "w0": dw0, "w1": dw1, "bias": db}

    base = {"x": x.astype(np.float64), "w0": w0.astype(np.float64),
            "w1": w1.astype(np.float64) if w1 is not None else None, "bias": bias.astype(np.float64)}
    # the oracle squeezes R' = 1 away for avg / max pooling (oracle.ri_forward)
    mm = m.reshape((n, cout, h, w)) if pool in ("avg", "max") else m.reshape((n, cout, -1, h, w))

    def fwd(vals):
        yy, aa = O.ri_forward(od, vals["x"], vals["w0"], vals["w1"], vals["bias"])
        if act == "relu":
            yy = np.maximum(yy, 0.0)
        return yy, aa

    def loss_of(name):
        def f(v):
            vals = dict(base)
            vals[name] = v
            return float((fwd(vals)[0] * mm).sum())
        return f

    y0, a0 = O.ri_forward(od, base["x"], base["w0"], base["w1"], base["bias"])

    def skip_of(name):
        # non-differentiable at the step: an argmax or a ReLU sign flips between x +- eps
        def skip(i, v, step):
            out = []
            for sgn in (1, -1):
                vals = dict(base)
                vv = v.copy()
                vv.reshape(-1)[i] += sgn * step
                vals[name] = vv
                out.append(O.ri_forward(od, vals["x"], vals["w0"], vals["w1"], vals["bias"]))
            if a0 is not None and any(not np.array_equal(o[1], a0) for o in out):
                return True
            if act == "relu" and any(not np.array_equal(o[0] > 0, y0 > 0) for o in out):
                return True
            return False
        return skip if (a0 is not None or act == "relu") else None

    for name in ("x", "w0", "w1", "bias"):
        if base[name] is None:
            continue
        gan = grads[name].double().cpu().numpy()
        err, used = fd.finite_diff_check(loss_of(name), base[name], gan, 1e-5, samples=50,
                                         seed=len(name), skip=skip_of(name))
        assert used >= min(30, base[name].size // 2), (name, used)
        assert err <= tol, (name, err)
