"""Pins for oracle/scalar.py against the paper's worked values and algebraic identities."""
import json
import math
import os

import numpy as np
import pytest

from oracle import scalar

pytestmark = pytest.mark.filterwarnings("ignore")


def _golden(golden_dir):
    with open(os.path.join(golden_dir, "spec_scalar_values.json")) as f:
        return json.load(f)


def test_spec_worked_values(golden_dir):
    g = _golden(golden_dir)
    for v in g["values"]:
        for m in v["m"]:
            if "t" in v:
                assert scalar.p_m(v["t"], m) == v["expect"], v["cite"]
            else:
                assert scalar.eps_m(v["gamma"], m) == v["expect"], v["cite"]
    for v in g["min_depth"]:
        assert scalar.min_depth(v["gamma"], v["tol"]) == v["expect"], v["cite"]
    for v in g["operator_error"]:
        gam = v["gamma"]
        mu = np.array([-1.0, -gam, -0.7, gam, 0.8, 1.0])
        assert abs(scalar.spectral_operator_error(mu, v["m"]) - v["expect"]) <= 1e-15, v["cite"]


def test_recurrence_equals_polynomial():
    """eq:ns_scalar_recurrence and eq:pm are two routes to 1-p_m(gamma)."""
    for gam in [1e-3, 0.05, 0.1, 0.25, 0.5, 0.9, 1.0]:
        for m in range(0, 25):
            assert abs(scalar.eps_m(gam, m) - (1.0 - scalar.p_m(gam, m))) <= 1e-12  # rounding amplified 1.5x/step in the linear regime


def test_fixed_point_factorisation():
    """lem:NSsign proof: f(t) - 1 = -1/2 (t-1)^2 (t+2); f maps (0,1] into (0,1]."""
    t = np.linspace(-1.5, 1.5, 3001)
    assert np.max(np.abs((scalar.p_step(t) - 1.0) - (-0.5 * (t - 1) ** 2 * (t + 2)))) <= 1e-15
    tp = np.linspace(1e-6, 1.0, 1001)
    ft = scalar.p_step(tp)
    assert np.all(ft > 0) and np.all(ft <= 1.0)


def test_sign_preservation_and_monotonicity():
    """lem:NSsign and prop:NSerr (p_m increasing on [0,1]); S:168 monotonicity."""
    t = np.linspace(-1.0, 1.0, 2001)
    t = t[np.abs(t) > 1e-12]
    for m in range(0, 9):
        pm = scalar.p_m(t, m)
        assert np.all(np.sign(pm) == np.sign(t))
        pos = scalar.p_m(np.linspace(0, 1, 1001), m)
        assert np.all(np.diff(pos) >= -5e-16)  # nondecreasing up to rounding near the fixed point 1
        assert np.max(np.abs(scalar.p_m(-t, m) + pm)) == 0.0  # odd


def test_quadratic_regime_bound():
    """eps_{m+1} <= 3/2 eps_m^2 (eq:ns_scalar_recurrence) for any gamma."""
    for gam in [0.01, 0.3, 0.5, 0.77]:
        for m in range(12):
            e0, e1 = scalar.eps_m(gam, m), scalar.eps_m(gam, m + 1)
            assert e1 <= 1.5 * e0 * e0 * (1 + 1e-15)


def test_near_linear_regime():
    """disc:spectral_compression: p_1(t) = 3/2 t + O(t^3) for small t."""
    for t in [1e-3, 1e-4, 1e-5]:
        assert abs(scalar.p_m(t, 1) - 1.5 * t) <= t ** 3


def test_predict_run_diagonal_matches_direct():
    """predict_run replays the loop on scalars: step j residual = ||diag(p_j(mu))^2 - I||_F."""
    mu = np.array([-0.9, -0.3, 0.2, 0.6, 1.0])
    steps, res, tr = scalar.predict_run(mu, 100, 1e-12, per_sqrt_d=False)
    for j in range(steps + 1):
        x = scalar.p_m(mu, j)
        assert abs(res[j] - math.sqrt(np.sum((x * x - 1) ** 2))) <= 1e-15
        assert abs(tr[j] - np.sum(x)) <= 1e-15
    assert res[steps] < 1e-12 and res[steps - 1] >= 1e-12
    # first step where eps_m(min|mu|) is tiny must be >= min_depth for tolerance in residual terms
    assert steps >= scalar.min_depth(0.2, 1e-6)


def test_min_depth_cap():
    with pytest.raises(ValueError):
        scalar.min_depth(1e-30, 1e-12, cap=10)
    with pytest.raises(ValueError):
        scalar.eps_m(0.0, 1)


def test_scaled_margin_closed_form():
    """gamma = min_i |lambda_i - s| / alpha (disc:spectral_compression P:484-490, divide form C1): the
    configs[3] spectrum edges give 0.05/1.05; the margin is the one prop:NSerr's bound uses, so the
    closed-form iterate's worst eigenvalue error equals eps_m(gamma) when an eigenvalue sits at the edge."""
    lam = np.array([-1.0, -0.05, 0.05, 0.3, 1.0])
    assert scalar.scaled_margin(lam, 0.0, 1.05) == 0.05 / 1.05
    assert abs(scalar.scaled_margin(lam, 0.1, 2.0) - 0.025) <= 1e-17
    g = scalar.scaled_margin(lam, 0.0, 1.05)
    mu = lam / 1.05
    for m in (1, 4, 9):
        assert abs(scalar.spectral_operator_error(mu, m) - scalar.eps_m(g, m)) <= 1e-15
