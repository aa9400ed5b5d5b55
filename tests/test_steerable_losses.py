"""SPEC:457-514 steerable regularisers -- the SPEC examples, on CPU tensors."""
import math

import pytest
import torch

import paper_2512_08888_b200 as P


def test_loss_mag_kats():
    b = P.SteerableBasis(torch.tensor([[[[3.0]]]]), torch.tensor([[[[1.0]]]]))
    assert P.loss_mag(b).item() == pytest.approx(4.0)          # (3 - 1)^2
    eq = P.SteerableBasis(torch.ones(2, 1, 3, 3), -torch.ones(2, 1, 3, 3))
    assert P.loss_mag(eq).item() == 0.0                         # equal norms


def test_loss_orth_kats():
    x = torch.randn(3, 2, 3, 3, dtype=torch.float64)
    assert P.loss_orth(P.SteerableBasis(x, x.clone())).item() == pytest.approx(1.0, abs=1e-6)
    gd = P.gaussian_derivative_basis(5, 1.0)
    assert P.loss_orth(gd).item() < 1e-20                       # odd symmetry: exactly orthogonal
    with pytest.raises(ValueError, match="eps must be positive"):
        P.loss_orth(gd, eps=0)


def test_total_loss_kat_and_gaussian_basis():
    gd = P.gaussian_derivative_basis(3, 0.8)
    assert abs(gd.f_x.norm().item() - 1) < 1e-12 and abs(gd.f_y.norm().item() - 1) < 1e-12
    assert torch.all(gd.f_x[..., :, 1] == 0)                    # zero column at x = 0
    assert P.total_loss(1.0, gd, 0.0, 0.0) == 1.0
    # ce=1, L_mag=4, L_orth=0.25, lambdas (0.5, 2) -> 3.5
    b = P.SteerableBasis(torch.tensor([[[[3.0, 0.0]]]]), torch.tensor([[[[0.5, math.sqrt(0.75) * 1.0]]]]))
    lm, lo = P.loss_mag(b).item(), P.loss_orth(b).item()
    assert P.total_loss(1.0, b, 0.5, 2.0).item() == pytest.approx(1 + 0.5 * lm + 2 * lo)
    with pytest.raises(ValueError, match="K must be odd"):
        P.gaussian_derivative_basis(4, 1.0)
