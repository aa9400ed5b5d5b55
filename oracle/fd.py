"""Central finite-difference verifier -- TEST INFRASTRUCTURE ONLY.

``finite_diff_check(f, point, grad, step)`` restates SPEC's ``finite_diff_check`` operation:
central differences (f(x + eps e_i) - f(x - eps e_i)) / (2 eps) in float64 at sampled
coordinates i, compared with an analytic gradient; returns the worst relative error,
normwise over the sample: max_i |fd_i - g_i| / max_i |g_i| (a per-coordinate ratio would
judge coordinates whose gradient is ~0 against round-off).  ``skip(i)`` may exclude coordinates where f is not differentiable
at the step (ties of a max pool, ReLU kinks), "at non-tied pixels".
"""
from __future__ import annotations

import numpy as np


def finite_diff_check(f, point: np.ndarray, grad: np.ndarray, step: float = 1e-5, coords=None,
                      samples: int = 50, seed: int = 0, skip=None):
    if step <= 0:
        raise ValueError("finite_diff_check: step must be positive")
    x = np.array(point, dtype=np.float64, copy=True)
    g = np.asarray(grad, dtype=np.float64).reshape(x.shape)
    flat, gflat = x.reshape(-1), g.reshape(-1)
    if coords is None:
        rng = np.random.default_rng(seed)
        coords = rng.choice(flat.size, size=min(samples, flat.size), replace=False)
    scale = max(np.abs(gflat[coords]).max(), np.finfo(np.float64).tiny)
    worst, used = 0.0, 0
    for i in coords:
        xi = flat[i]
        flat[i] = xi + step
        fp = f(x)
        flat[i] = xi - step
        fm = f(x)
        flat[i] = xi
        if skip is not None and skip(i, x, step):
            continue
        fd = (fp - fm) / (2 * step)
        worst = max(worst, abs(fd - gflat[i]) / scale)
        used += 1
    return worst, used
