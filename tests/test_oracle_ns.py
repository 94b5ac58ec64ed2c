"""Pins for oracle/ns.py, oracle/jacobi.py and oracle/closed_form.py.

Each test checks the oracle against something other than itself: closed forms from
the generator's known Q (thm:generic proof P:308-312), the scalar recurrence
(prop:NSerr), the paper's invariants (prop:exact), LAPACK (third path), the DFT
spectrum of the periodic Laplacian, and 50-digit mpmath brute force for d <= 16.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import checks, closed_form, jacobi, ns, scalar
import workloads


# ----------------------------------------------------------------- special cases
def test_diagonal_consistency():
    """diagonal H -> X_m = diag(p_m((h_ii - s)/alpha)) exactly up to rounding."""
    h = np.array([-3.0, -1.0, -0.25, 0.5, 2.0, 4.0])
    s, alpha = 0.1, 4.2
    for m in range(0, 7):
        out = ns.ns_reflector(np.diag(h), s, alpha, 3, m, 0.0)
        expect = scalar.p_m((h - s) / alpha, m)
        assert out["steps"] == m and out["flags"] & ns.MAX_STEPS
        assert np.max(np.abs(np.diag(out["R"]) - expect)) <= 4e-16
        assert np.max(np.abs(out["R"] - np.diag(np.diag(out["R"])))) == 0.0


def test_fixed_points_and_zero():
    """diag(-1,1) is a fixed point; A = 0 stays 0 (never converges)."""
    out = ns.ns_reflector(np.diag([-1.0, 1.0]), 0.0, 1.0, 1, 5, 1e-12)
    assert out["steps"] == 0 and out["flags"] == ns.CONVERGED and out["cert"] == 1
    assert np.array_equal(out["R"], np.diag([-1.0, 1.0]))
    z = ns.ns_reflector(np.zeros((4, 4)), 0.0, 1.0, 0, 7, 1e-12)
    assert z["steps"] == 7 and z["flags"] & ns.MAX_STEPS and np.all(z["R"] == 0)
    assert z["flags"] == ns.MAX_STEPS | ns.INDEX_MISMATCH and z["cert"] == 2 and z["residual"] == 2.0
    # s outside the spectrum: k = 0 or d gives +-I (C8)
    hp = np.diag([1.0, 2.0, 3.0])
    up = ns.ns_reflector(hp, 0.0, 3.0, 0, 100, 1e-12)
    assert up["cert"] == 0 and np.max(np.abs(up["R"] - np.eye(3))) < 1e-13
    dn = ns.ns_reflector(hp, 10.0, 9.0, 3, 100, 1e-12)
    assert dn["cert"] == 3 and np.max(np.abs(dn["R"] + np.eye(3))) < 1e-13


def test_spec_exact_reflector_examples(golden_dir):
    with open(os.path.join(golden_dir, "spec_scalar_values.json")) as f:
        g = json.load(f)
    for ex in g["exact_reflector"]:
        R, w = jacobi.exact_reflector(np.diag(ex["H_diag"]), ex["k"])
        assert np.max(np.abs(R - np.diag(ex["expect_diag"]))) <= 1e-15, ex["cite"]


# ----------------------------------------------------------------- closed forms
@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4])
def test_cfg0_iterates_match_closed_form(seed):
    """X_m (oracle loop) == Q diag(p_m(mu)) Q^T (thm:generic proof) for every m up to convergence."""
    p = workloads.cfg0_controlled(seed)
    for m in range(0, 10):
        X = ns.ns_reflector(p.H, p.s, p.alpha, p.k, m, 0.0)["R"]
        Xcf = closed_form.iterate_explicit_q(p.Q, p.lam, p.s, p.alpha, m)
        assert np.max(np.abs(X - Xcf)) <= 2e-14, m


@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4])
def test_cfg0_full_run(seed):
    """cfg0: steps == scalar-recurrence prediction, R == closed form == Jacobi I-2P_3, invariants."""
    p = workloads.cfg0_controlled(seed)
    out = ns.ns_reflector(p.H, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode)
    mu = (p.lam - p.s) / p.alpha
    steps_pred, res_pred, _ = scalar.predict_run(mu, p.max_steps, p.tol, False)
    assert out["steps"] == steps_pred
    assert out["flags"] == ns.CONVERGED and out["cert"] == p.k
    R_cf = closed_form.reflector_explicit_q(p.Q, p.lam, p.s)
    R_eig, w = jacobi.exact_reflector(p.H, p.k)
    assert checks.frob_per_sqrt_d(out["R"], R_cf) <= 1e-14
    assert checks.frob_per_sqrt_d(out["R"], R_eig) <= 1e-13
    inv = checks.reflector_invariants(out["R"], p.H, p.k)
    assert inv["square"] < 1e-13 and inv["symmetry"] == 0.0 and inv["commutator"] < 1e-13 and inv["trace"] < 1e-12
    assert np.max(np.abs(np.sort(p.lam) - w)) <= 1e-13


def test_gapped_operator_bound():
    """prop:NSerr eq:NSoperr: ||p_m(A) - sgn A||_2 <= eps_m(gamma), equality with an eigenvalue at +-gamma."""
    rng = np.random.default_rng(7)
    d = 24
    for gam in [0.05, 0.1, 0.25, 0.5]:
        mags = rng.uniform(gam, 1.0, d)
        mags[0] = gam
        mu = mags * np.where(np.arange(d) % 3 == 0, -1.0, 1.0)
        Q = workloads.haar_q(rng, d)
        A = 0.5 * ((Q * mu) @ Q.T + ((Q * mu) @ Q.T).T)
        S = closed_form.reflector_explicit_q(Q, mu, 0.0)
        for m in range(0, 9):
            X = ns.ns_fixed_depth(A, 1.0, m)
            err = np.linalg.norm(X - S, 2)
            assert err <= scalar.eps_m(gam, m) + 1e-9
            assert abs(err - scalar.eps_m(gam, m)) <= 1e-12


def test_shift_independence_cfg1():
    """prop:exact: the three cfg1 shifts give the same exact reflector; the midpoint needs strictly
    fewer steps than either off-midpoint shift (prop:mid, SURVEY EXP-2c)."""
    probs = workloads.cfg1_batched(seed=0, first=0, count=2, d=64)
    for b in range(2):
        trio = probs[3 * b:3 * b + 3]
        outs = [ns.ns_reflector(p.H, p.s, p.alpha, p.k, p.max_steps, p.tol) for p in trio]
        for o, p in zip(outs, trio):
            assert o["flags"] == ns.CONVERGED and o["cert"] == p.k
            mu = (p.lam - p.s) / p.alpha
            assert o["steps"] == scalar.predict_run(mu, 100, 1e-12, False)[0]
        assert checks.frob_per_sqrt_d(outs[0]["R"], outs[1]["R"]) <= 1e-13
        assert checks.frob_per_sqrt_d(outs[0]["R"], outs[2]["R"]) <= 1e-13
        assert outs[0]["steps"] < min(outs[1]["steps"], outs[2]["steps"])


def test_householder_closed_form_and_generator():
    """Q = H_1...H_n: orthogonal; generator's H = Q diag(lam) Q^T; closed-form columns == explicit."""
    lam, Vh = workloads.householder_spectrum(1, 256, 16, 0.05, 8)
    Q = closed_form.householder_apply(Vh, np.eye(256))
    assert np.max(np.abs(Q.T @ Q - np.eye(256))) <= 1e-14
    H = workloads.householder_form_numpy(Vh, lam)
    assert np.max(np.abs(H - (Q * lam) @ Q.T)) <= 1e-14
    cols = [0, 5, 77, 255]
    Rc = closed_form.householder_reflector_columns(Vh, lam, 0.0, cols)
    R = closed_form.reflector_explicit_q(Q, lam, 0.0)
    assert np.max(np.abs(Rc - R[:, cols])) <= 1e-14


def test_householder_iterate_columns_match_ns_loop():
    """thm:generic: the m-step iterate of the NS loop on H = Q diag(lam) Q^T equals
    Q diag(p_m((lam - s)/alpha)) Q^T; the Householder column routine is that closed form (two routes:
    matrix products vs. scalar polynomial + reflector applications)."""
    lam, Vh = workloads.householder_spectrum(3, 200, 12, 0.05, 10)
    H = workloads.householder_form_numpy(Vh, lam)
    cols = [0, 3, 99, 199]
    for m in (0, 1, 3, 7):
        Xm = ns.ns_fixed_depth(H - 0.1 * np.eye(200), 1.2, m)
        Xc = closed_form.householder_iterate_columns(Vh, lam, 0.1, 1.2, m, cols)
        assert np.max(np.abs(Xm[:, cols] - Xc)) <= 1e-13, m
    # m large: the closed-form iterate is the reflector (prop:exact)
    Xc = closed_form.householder_iterate_columns(Vh, lam, 0.1, 1.2, 40, cols)
    assert np.max(np.abs(Xc - closed_form.householder_reflector_columns(Vh, lam, 0.1, cols))) <= 1e-13


def test_timed_ns_steps_is_the_ns_loop():
    """The cpu_baseline helper runs the same arithmetic as ns_reflector: after n fixed steps its iterate is
    bitwise ns_reflector's (tol = 0, max_steps = n, reading C5)."""
    p = workloads.cfg0_controlled(seed=4, d=96, k=5)
    for n in (1, 3):
        t, threads, X = ns.timed_ns_steps(p.H, p.s, p.alpha, n, return_iterate=True)
        o = ns.ns_reflector(p.H, p.s, p.alpha, p.k, n, 0.0)
        assert o["steps"] == n and np.array_equal(X, o["R"])
        assert t >= 0.0 and threads >= 1


def test_householder_fast_formation():
    """The WY formation used for large-d inputs equals the inside-out rank-2 recipe (C13)."""
    lam, Vh = workloads.householder_spectrum(1, 300, 20, 0.05, 16)
    H1 = workloads.householder_form_numpy(Vh, lam)
    H2 = workloads.householder_form_fast(Vh, lam)
    assert np.array_equal(H2, H2.T)
    assert np.max(np.abs(H1 - H2)) <= 1e-14


def test_cfg3_recipe_reduced_size():
    """cfg3 recipe at d=1024, k=64 (C13): steps == prediction (both tol readings, C3); R == closed form."""
    p = workloads.cfg3_dense(d=1024, k=64)
    out = ns.ns_reflector(p.H, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode, trace_residuals=True)
    mu = (p.lam - p.s) / p.alpha
    steps_pred, res_pred, _ = scalar.predict_run(mu, 100, 1e-10, True)
    assert out["steps"] == steps_pred and out["cert"] == 64 and out["flags"] == ns.CONVERGED
    # residual history follows the eigenvalue-wise closed form until the rounding floor
    for j in range(out["steps"]):
        assert abs(out["hist_residual"][j] - res_pred[j]) <= 1e-12 * max(1.0, res_pred[j]) + 1e-13
    cols = np.arange(0, 1024, 37)
    Rc = closed_form.householder_reflector_columns(p.Vh, p.lam, 0.0, cols)
    assert np.max(np.abs(out["R"][:, cols] - Rc)) <= 1e-13


# ----------------------------------------------------------------- Jacobi vs LAPACK (third path)
@pytest.mark.parametrize("d", [5, 16, 64, 200])
def test_jacobi_vs_lapack(d):
    rng = np.random.default_rng(d)
    A = rng.standard_normal((d, d))
    A = 0.5 * (A + A.T)
    w, V, sweeps = jacobi.jacobi_eigh(A)
    assert sweeps <= 60
    assert np.max(np.abs(w - np.linalg.eigvalsh(A))) <= 1e-12 * max(1.0, np.max(np.abs(w)))
    assert np.max(np.abs((V * w) @ V.T - A)) <= 1e-10
    assert np.max(np.abs(V.T @ V - np.eye(d))) <= 1e-10


# ----------------------------------------------------------------- Allen–Cahn closed form (u = 0)
def test_allen_cahn_u0_dft_closed_form():
    """u = 0: H = eps^2 L_h - I, periodic 5-point stencil, spectrum
    eps^2 (4/h^2)(sin^2(pi p/n) + sin^2(pi q/n)) - 1; k=5 gap; R = I - 2 P_5 with P_5 the
    projector onto the grid samples of {1, cos2pi x, sin2pi x, cos2pi y, sin2pi y}."""
    n = 16
    prob = workloads.cfg2_allen_cahn(u=np.zeros(n * n), n=n)
    H = prob.H
    h = 1.0 / n
    pq = np.arange(n)
    S2 = np.sin(np.pi * pq / n) ** 2
    lam_dft = np.sort((0.04 ** 2 * 4 / h ** 2 * (S2[:, None] + S2[None, :])).reshape(-1) - 1.0)
    w, V, _ = jacobi.jacobi_eigh(H)
    assert np.max(np.abs(w - lam_dft)) <= 1e-12
    s = jacobi.midpoint_shift(w, 5)
    alpha = workloads.configs.gershgorin_alpha(H, s)
    # Gershgorin shortcut: max|H_ii - s| + 4 eps^2/h^2
    assert abs(alpha - (np.max(np.abs(np.diag(H) - s)) + 4 * 0.04 ** 2 / h ** 2)) <= 1e-12
    x = np.arange(n) / n
    X, Y = np.meshgrid(x, x, indexing="xy")
    B = np.stack([np.ones_like(X), np.cos(2 * np.pi * X), np.sin(2 * np.pi * X),
                  np.cos(2 * np.pi * Y), np.sin(2 * np.pi * Y)], axis=-1).reshape(n * n, 5)
    Qb, _ = np.linalg.qr(B)
    R_cf = np.eye(n * n) - 2 * Qb @ Qb.T
    R_eig = jacobi.exact_reflector_from_eig(V, 5)
    assert checks.frob_per_sqrt_d(R_eig, R_cf) <= 1e-13
    out = ns.ns_reflector(H, s, alpha, 5, 100, 1e-12)
    assert out["flags"] == ns.CONVERGED and out["cert"] == 5
    assert checks.frob_per_sqrt_d(out["R"], R_cf) <= 1e-13
    steps_pred = scalar.predict_run((lam_dft - s) / alpha, 100, 1e-12, False)[0]
    assert abs(out["steps"] - steps_pred) <= 1


def test_allen_cahn_seeded_field():
    """Seeded field is normalised (max|u| = 1), smooth (8 modes, |k|<=4) and H is symmetric."""
    u = workloads.configs.allen_cahn_field(0, n=16)
    assert abs(np.max(np.abs(u)) - 1.0) <= 1e-15
    H = workloads.configs.allen_cahn_hessian(u, n=16)
    assert np.array_equal(H, H.T)
    F = np.fft.fft2(u.reshape(16, 16))
    kk = np.fft.fftfreq(16, 1 / 16)
    mask = (np.abs(kk)[:, None] > 4) | (np.abs(kk)[None, :] > 4)
    assert np.max(np.abs(F[mask])) <= 1e-12


# ----------------------------------------------------------------- brute force, d <= 16
def test_mpmath_brute_force_tiny():
    """north_star: brute force on d <= 16 -- 50-digit NS loop and mpmath eigsy reflector."""
    mp = pytest.importorskip("mpmath")
    mp.mp.dps = 50
    p = workloads.cfg0_controlled(seed=3, d=12, k=3)
    out = ns.ns_reflector(p.H, p.s, p.alpha, p.k, 100, 1e-12)
    d = p.d
    Hm = mp.matrix(p.H.tolist())
    X = (Hm - mp.mpf(float(p.s)) * mp.eye(d)) / mp.mpf(float(p.alpha))
    for _ in range(out["steps"]):
        X = 1.5 * X - 0.5 * (X * (X * X))
    Xn = np.array(X.tolist(), dtype=np.float64)
    assert np.max(np.abs(Xn - out["R"])) <= 1e-14
    E, Qm = mp.eigsy(Hm)
    order = sorted(range(d), key=lambda i: E[i])
    Qk = mp.matrix(d, p.k)
    for c, i in enumerate(order[:p.k]):
        for r in range(d):
            Qk[r, c] = Qm[r, i]
    Rm = mp.eye(d) - 2 * (Qk * Qk.T)
    Rn = np.array(Rm.tolist(), dtype=np.float64)
    R_eig, _ = jacobi.exact_reflector(p.H, p.k)
    assert np.max(np.abs(Rn - R_eig)) <= 1e-14
    assert np.max(np.abs(Rn - out["R"])) <= 1e-14


# ----------------------------------------------------------------- flags
def test_flags_scaling_and_mismatch():
    """alpha far below ||H - sI||_2 -> residual rise (SCALING_SUSPECT) / non-finite; wrong k -> INDEX_MISMATCH."""
    p = workloads.cfg0_controlled(seed=0)
    bad = ns.ns_reflector(p.H, p.s, p.alpha / 4.0, p.k, 100, 1e-12)
    assert bad["flags"] & (ns.SCALING_SUSPECT | ns.NONFINITE)
    mis = ns.ns_reflector(p.H, p.s, p.alpha, p.k + 1, 100, 1e-12)
    assert mis["flags"] == ns.CONVERGED | ns.INDEX_MISMATCH and mis["cert"] == p.k
    nanH = p.H.copy()
    nanH[3, 5] = nanH[5, 3] = np.nan
    nf = ns.ns_reflector(nanH, p.s, p.alpha, p.k, 100, 1e-12)
    assert nf["flags"] & ns.NONFINITE and nf["steps"] == 0
    # shift on the spectrum: s = lambda_3 exactly -> trace half-integer-ish or residual stuck
    ls = np.sort(p.lam)
    on = ns.ns_reflector(p.H, ls[2], p.alpha, p.k, 60, 1e-12)
    assert on["flags"] & ns.MAX_STEPS


def test_round_half_away():
    assert ns.round_half_away(2.5) == 3 and ns.round_half_away(-2.5) == -3
    assert ns.round_half_away(2.4999) == 2 and ns.round_half_away(0.0) == 0
