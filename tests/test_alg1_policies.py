"""Pins for Algorithm 1's shift policies and admissibility stop (oracle/outer.py; alg:ssr P:653-701,
prop:reuse_refresh P:587-651, prop:exact P:147-165).  CPU only."""

import numpy as np
import pytest

import workloads
from oracle import outer


def test_choose_shift_hand_values():
    """alg:ssr step 4 on hand-computed endpoint pairs (lambda_k, lambda_k+1) = (1, 3): midpoint 2; damped blend
    beta s_prev + (1 - beta) mid clipped to [1 + kappa 2, 3 - kappa 2]; reuse while the margin exceeds tau."""
    cs = outer.choose_shift
    assert cs("midpoint", 1.0, 3.0, 2.9) == (2.0, True)
    assert cs("damped", 1.0, 3.0, None) == (2.0, True)                     # n = 0: no previous shift
    assert cs("damped", 1.0, 3.0, 2.9, damp=0.5, clip=0.25) == (2.45, False)   # inside [1.5, 2.5]
    assert cs("damped", 1.0, 3.0, 10.0, damp=0.5, clip=0.25) == (2.5, False)   # 6.0 clipped to the top
    assert cs("damped", 1.0, 3.0, -10.0, damp=0.5, clip=0.25) == (1.5, False)  # -4.0 clipped to the bottom
    assert cs("damped", 1.0, 3.0, 2.9, damp=0.0, clip=0.1) == (2.0, False)     # beta = 0: the midpoint
    assert cs("damped", 1.0, 3.0, 2.9, damp=0.9, clip=0.5) == (2.0, False)     # kappa = 1/2: the midpoint
    assert cs("reuse_refresh", 1.0, 3.0, 2.5, reuse_margin=0.4) == (2.5, False)   # margin 0.5 > 0.4: keep
    assert cs("reuse_refresh", 1.0, 3.0, 2.5, reuse_margin=0.6) == (2.0, True)    # margin 0.5 <= 0.6: refresh
    assert cs("reuse_refresh", 1.0, 3.0, 3.5, reuse_margin=0.0) == (2.0, True)    # left the gap: refresh
    assert cs("reuse_refresh", 1.0, 3.0, 1.2, reuse_margin=0.0) == (1.2, False)


def _scalar_diag_run(x0, k, m, eta, iters, policy, damp=0.5, clip=0.25, tau=0.0):
    """Q = I: every matrix in alg:ssr is diagonal, so one iteration is scalar arithmetic per coordinate --
    mu_i = 3 x_i^2 + c_i, g_i = x_i^3 + c_i x_i, filter value p^m((mu_i - s)/alpha) with the scalar NS map
    p(t) = 1.5 t - 0.5 t^3 (eq:pm P:380-384), x_i <- x_i - eta f_i g_i.  Written without matrices."""
    x = list(x0)
    d = len(x)
    s_prev = None
    shifts = []
    for _ in range(iters):
        c = [-1.0 if i < k else 1.0 for i in range(d)]
        mu = [3 * x[i] ** 2 + c[i] for i in range(d)]
        g = [x[i] ** 3 + c[i] * x[i] for i in range(d)]
        lk, lk1 = sorted(mu)[k - 1], sorted(mu)[k]
        mid = (lk + lk1) / 2
        if s_prev is None or policy == "midpoint":
            s = mid
        elif policy == "damped":
            s = min(max(damp * s_prev + (1 - damp) * mid, lk + clip * (lk1 - lk)), lk1 - clip * (lk1 - lk))
        else:
            s = s_prev if min(s_prev - lk, lk1 - s_prev) > tau else mid
        alpha = max(abs(v - s) for v in mu)
        f = []
        for i in range(d):
            t = (mu[i] - s) / alpha
            for _ in range(m):
                t = 1.5 * t - 0.5 * t ** 3
            f.append(t)
        x = [x[i] - eta * f[i] * g[i] for i in range(d)]
        shifts.append(s)
        s_prev = s
    return np.array(x), shifts


@pytest.mark.parametrize("policy,kw", [("midpoint", {}), ("damped", dict(damp=0.6, clip=0.2)),
                                       ("reuse_refresh", dict(reuse_margin=0.3))])
def test_policies_on_diagonal_model(policy, kw):
    """Q = I (d = 3, k = 1): three iterations of the matrix oracle equal the scalar per-coordinate
    computation (a transposed Q, a wrong NS coefficient, a sign in the update or a wrong policy branch fails)."""
    x0 = [0.7, -0.4, 0.25]
    r = outer.run(np.eye(3), 1, np.array(x0), 2, 0.3, 3, 0.0, policy=policy, **kw)
    tau = kw.get("reuse_margin", 0.0)
    xs, shifts = _scalar_diag_run(x0, 1, 2, 0.3, 3, policy, kw.get("damp", 0.5), kw.get("clip", 0.25), tau)
    assert r["iters"] == 3 and r["stop_reason"] == outer.STOP_BUDGET
    assert np.max(np.abs(r["x"] - xs)) <= 1e-14
    assert np.max(np.abs(np.array(r["shifts"]) - np.array(shifts))) <= 1e-14


def test_admissibility_stop_hand_case():
    """Step 8 "stop if the shift ceases to be admissible" with prop:reuse_refresh's test m_hat > eps:
    Q = I, k = 1, x0 = (1/2, 1/4): mu = (-1/4, 19/16) (exact in binary), midpoint 15/32, margin 23/32.
    eps = 0.7 proceeds, eps = 23/32 stops before any update."""
    x0 = np.array([0.5, 0.25])
    r = outer.run(np.eye(2), 1, x0, 2, 0.1, 1, 0.0, eps=0.7)
    assert r["stop_reason"] == outer.STOP_BUDGET and r["iters"] == 1 and r["shifts"] == [15 / 32]
    r = outer.run(np.eye(2), 1, x0, 2, 0.1, 5, 0.0, eps=23 / 32)
    assert r["stop_reason"] == outer.STOP_INADMISSIBLE and r["iters"] == 0 and r["refreshes"] == 0
    assert np.array_equal(r["x"], x0)


def test_gap_closing_stops_inadmissible():
    """A run whose target gap closes: Q = I, k = 1, c = (-1, +1), mu = (3 y1^2 - 1, 3 y2^2 + 1).  The two
    values cross where 3 y1^2 - 1 = 3 y2^2 + 1; with eps = 0.05 the run stops (inadmissible) once the
    estimated gap falls to 2 eps, i.e. before the crossing.  Checked against the scalar gap."""
    x0 = np.array([0.9, 0.1])   # mu = (1.43, 1.03): sorted endpoints (1.03, 1.43), gap 0.4
    r = outer.run(np.eye(2), 1, x0, 0, 0.05, 200, 0.0, eps=0.05)
    assert r["stop_reason"] == outer.STOP_INADMISSIBLE
    y1, y2 = r["x"]
    gap = abs((3 * y1 * y1 - 1) - (3 * y2 * y2 + 1))
    assert gap <= 0.1 + 1e-15
    assert r["iters"] >= 1


@pytest.mark.parametrize("kw", [dict(policy="damped", damp=0.7, clip=0.1), dict(policy="damped", damp=0.3, clip=0.4),
                                dict(policy="reuse_refresh", reuse_margin=0.05),
                                dict(policy="reuse_refresh", reuse_margin=0.5)])
def test_exact_reflector_is_shift_independent(kw):
    """prop:exact: every admissible shift gives the same exact reflector, so with m = 0 the
    trajectories under the damped and reuse/refresh policies equal the midpoint run bit for bit, while the
    shift histories differ (the policies are exercised)."""
    Q, ks, starts = workloads.rotated_quartic_scan(d=16, ks=(1, 4), n_starts=2, radius=2.0)
    differ = 0
    for k in ks:
        for x0 in starts:
            a = outer.run(Q, k, x0, 0, 0.2, 60, 1e-10)
            b = outer.run(Q, k, x0, 0, 0.2, 60, 1e-10, **kw)
            if outer.STOP_INADMISSIBLE in (a["stop_reason"], b["stop_reason"]):
                continue   # a closing gap: when the margin rounds away depends on the shift's position
            assert a["iters"] == b["iters"] and a["stop_reason"] == b["stop_reason"]
            assert np.array_equal(a["x"], b["x"])
            differ += int(a["shifts"] != b["shifts"])
    assert differ > 0


@pytest.mark.parametrize("kw", [dict(policy="midpoint"), dict(policy="damped", damp=0.5, clip=0.2),
                                dict(policy="reuse_refresh", reuse_margin=0.1)])
def test_policies_converge_locally(kw):
    """thm:discrete: with an admissible shift policy and an accurate filter (m = 6) runs started
    near the index-k saddle converge to it.  Under reuse/refresh with a small threshold the shift is reused
    (fewer refreshes than iterations)."""
    Q, ks, starts = workloads.rotated_quartic_scan(d=16, ks=(1, 4), n_starts=3, radius=0.1)
    for k in ks:
        for x0 in starts:
            r = outer.run(Q, k, x0, 6, 0.2, 500, 1e-10, **kw)
            assert r["success"] and r["stop_reason"] == outer.STOP_GRAD and np.linalg.norm(r["x"]) < 1e-9
            if kw["policy"] == "reuse_refresh":
                assert r["refreshes"] < r["iters"]
            if kw["policy"] == "midpoint":
                assert r["refreshes"] == r["iters"]
