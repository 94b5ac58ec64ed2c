"""N1 (shift/scale setup) and N3 (filter variants): oracle pins on CPU, and the C library's
host-only certificate against the oracle's transcription of prop:reuse_refresh."""
import numpy as np
import pytest

from oracle import closed_form, setup, scalar
import workloads


def test_inf_norm_pins():
    # diagonal: max |h_ii - s| ; Gershgorin: >= spectral norm; equals numpy's inf-norm
    assert setup.inf_norm_shifted(np.diag([-3.0, 1.0, 2.5]), 0.5) == 3.5
    rng = np.random.default_rng(3)
    for d in (5, 40, 130):
        A = rng.standard_normal((d, d))
        A = 0.5 * (A + A.T)
        s = float(rng.uniform(-1, 1))
        v = setup.inf_norm_shifted(A, s)
        assert v >= np.linalg.norm(A - s * np.eye(d), 2) - 1e-12
        assert abs(v - np.linalg.norm(A - s * np.eye(d), np.inf)) <= 1e-12 * v


def test_certificate_pins():
    c = setup.shift_certificate(-1.0, 1.0, 0.1, 0.0, 0.5)
    assert c["margin_hat"] == 1.0 and c["admissible"] and abs(c["margin_lb"] - 0.9) < 1e-15
    assert c["reuse_ok"] and abs(c["reuse_margin_lb"] - 0.4) < 1e-15 and c["midpoint"] == 0.0
    assert not setup.shift_certificate(-1.0, 1.0, 0.1, 0.0, 0.95)["reuse_ok"]
    assert not setup.shift_certificate(-1.0, 1.0, 1.0, 0.0)["admissible"]      # m_hat == eps: not strict
    assert not setup.shift_certificate(0.0, 0.1, 0.06, 0.05)["midpoint_ok"]
    # brute force: any true endpoints within eps of the estimates, drifted by <= delta, keep s inside
    rng = np.random.default_rng(0)
    for _ in range(2000):
        lk, lk1 = sorted(rng.uniform(-1, 1, 2))
        eps, delta = rng.uniform(0, 0.2, 2)
        s = rng.uniform(lk - 0.1, lk1 + 0.1)
        c = setup.shift_certificate(lk, lk1, eps, s, delta)
        tk = lk + rng.uniform(-eps, eps)
        tk1 = lk1 + rng.uniform(-eps, eps)
        if c["admissible"]:
            assert tk < s < tk1 and min(s - tk, tk1 - s) >= c["margin_lb"] - 1e-15
        if c["reuse_ok"]:
            nk, nk1 = tk + rng.uniform(-delta, delta), tk1 + rng.uniform(-delta, delta)
            assert nk < s < nk1 and min(s - nk, nk1 - s) >= c["reuse_margin_lb"] - 1e-15


def test_c_certificate_matches_oracle():
    from paper_2605_24840_b200 import build
    build.build()
    import paper_2605_24840_b200 as nsr
    rng = np.random.default_rng(1)
    for _ in range(500):
        lk, lk1 = sorted(rng.uniform(-2, 2, 2))
        eps, delta = rng.uniform(0, 0.5, 2)
        s = rng.uniform(-2.5, 2.5)
        a = setup.shift_certificate(lk, lk1, eps, s, delta)
        b = nsr.ns_shift_certificate(lk, lk1, eps, s, delta)
        assert a == b


def test_filter_oracle_pins():
    """Odd cubic filters: diagonal exactness and the closed form Q diag(phi^m(mu)) Q^T; NS is (1.5, -0.5)."""
    h = np.array([-0.9, -0.2, 0.3, 0.7])
    for (a, b) in ((1.5, -0.5), (1.875, -0.875), (1.0, 0.0)):
        for m in (0, 2, 4, 6):
            X = setup.filter_fixed_depth(np.diag(h), 0.1, 1.0, m, a, b)
            assert np.max(np.abs(np.diag(X) - setup.filter_scalar(h - 0.1, m, a, b))) <= 1e-15
    assert np.array_equal(setup.filter_scalar(0.5, 3, 1.5, -0.5), scalar.p_m(0.5, 3))
    p = workloads.cfg0_controlled(seed=1)
    for m in (2, 4, 6):
        X = setup.filter_fixed_depth(p.H, p.s, p.alpha, m, 1.875, -0.875)
        mu = (p.lam - p.s) / p.alpha
        Xcf = closed_form.spectral_matrix(p.Q, setup.filter_scalar(mu, m, 1.875, -0.875))
        assert np.max(np.abs(X - Xcf)) <= 1e-13
    # sign preservation of the alternative filter on [-1, 1] (eq:signpreserving)
    t = np.linspace(-1, 1, 2001)
    t = t[t != 0]
    assert np.all(np.sign(setup.filter_scalar(t, 5, 1.875, -0.875)) == np.sign(t))


# ------------------------------------------------------------------ N2: Algorithm 1 oracle pins
def test_rotated_quartic_model_pins():
    """Gradient and Hessian eigenvalues of the rotated quartic: finite differences,
    origin is a critical point with Morse index k, Hessian eigenvalues mu = 3y^2 + c."""
    from oracle import outer
    Q, ks, starts = workloads.rotated_quartic_scan(d=8, ks=(3,), n_starts=2)
    k = 3
    c = np.where(np.arange(8) < k, -1.0, 1.0)
    E = lambda x: 0.25 * np.sum((Q.T @ x) ** 4) + 0.5 * np.sum(c * (Q.T @ x) ** 2)  # noqa: E731
    x = starts[0]
    g, mu = outer.gradient_and_mu(Q, k, x)
    h = 1e-6
    fd = np.array([(E(x + h * e) - E(x - h * e)) / (2 * h) for e in np.eye(8)])
    assert np.max(np.abs(fd - g)) <= 1e-5 * max(1.0, np.linalg.norm(g))   # S:481 tolerance
    y = Q.T @ x
    H = Q @ np.diag(3 * y * y + c) @ Q.T
    assert np.max(np.abs(np.sort(np.linalg.eigvalsh(H)) - np.sort(mu))) <= 1e-12
    g0, mu0 = outer.gradient_and_mu(Q, k, np.zeros(8))
    assert np.all(g0 == 0) and np.sum(mu0 < 0) == k


def test_alg1_exact_reflector_converges_locally():
    """thm:discrete / SPEC S:448: matched-index runs from within radius 0.1 converge to the origin
    (index-k saddle) with the exact reflector and with NS depth 6."""
    from oracle import outer
    Q, ks, starts = workloads.rotated_quartic_scan(d=16, ks=(1, 4), n_starts=3, radius=0.1)
    for k in ks:
        for x0 in starts:
            for m in (0, 6):
                r = outer.run(Q, k, x0, m, 0.2, 500, 1e-10)
                assert r["success"] and np.linalg.norm(r["x"]) < 1e-9, (k, m, r["iters"])


def test_inertia_matches_sylvester_ldl():
    """#{lambda < s} from the oracle's Jacobi eigenvalues equals the inertia of the LDL^T factorisation of
    H - sI (Sylvester's law of inertia: negative eigenvalues of the block-diagonal D), a route that never
    forms eigenvalues."""
    import scipy.linalg
    from oracle import jacobi
    rng = np.random.default_rng(5)
    for d in (7, 40, 90):
        A = rng.standard_normal((d, d))
        A = 0.5 * (A + A.T)
        w, _, _ = jacobi.jacobi_eigh(A)
        for s in rng.uniform(w[0] - 0.5, w[-1] + 0.5, 6):
            _, D, _ = scipy.linalg.ldl(A - s * np.eye(d))
            neg = int(np.count_nonzero(np.linalg.eigvalsh(D) < 0))   # D: 1x1 and 2x2 blocks
            assert setup.inertia(w, s) == neg


def test_shift_bisect_pins():
    """The bisection on exact counts: the returned brackets contain lambda_k and lambda_k+1, the shift lies
    strictly inside the gap with margin >= gap/2 - 2 eps, and eps <= rel_eps * estimated gap; multiple
    eigenvalues (the Allen-Cahn u = 0 Hessian's 4-fold lambda_2..5, k = 5) and brute force on random spectra."""
    # Allen-Cahn u = 0 on the 64x64 grid: closed-form spectrum (DFT of the periodic 5-point stencil)
    n, eps2, h = 64, 0.04 ** 2, 1.0 / 64
    p, q = np.meshgrid(np.arange(n), np.arange(n))
    lam = np.sort((eps2 * 4 / h ** 2 * (np.sin(np.pi * p / n) ** 2 + np.sin(np.pi * q / n) ** 2) - 1.0).ravel())
    r = setup.shift_bisect(lambda s: setup.inertia(lam, s), 5, -60.0, 60.0, 0.05, 200)
    assert r["ok"] and lam[4] < r["s"] < lam[5]
    assert r["lam_k_lo"] <= lam[4] <= r["lam_k_hi"] and r["lam_k1_lo"] <= lam[5] <= r["lam_k1_hi"]
    gap_hat = 0.5 * (r["lam_k1_lo"] + r["lam_k1_hi"]) - 0.5 * (r["lam_k_lo"] + r["lam_k_hi"])
    assert r["eps"] <= 0.05 * gap_hat
    assert min(r["s"] - lam[4], lam[5] - r["s"]) >= 0.5 * gap_hat - 2 * r["eps"]
    rng = np.random.default_rng(9)
    for _ in range(300):
        d = int(rng.integers(2, 60))
        lam = np.sort(rng.uniform(-3, 3, d))
        k = int(rng.integers(1, d))
        if lam[k] - lam[k - 1] < 1e-6:
            continue
        r = setup.shift_bisect(lambda s: setup.inertia(lam, s), k, -4.0, 4.0, 0.1, 400)
        assert r["ok"] and lam[k - 1] < r["s"] < lam[k]
        assert r["lam_k_lo"] <= lam[k - 1] <= r["lam_k_hi"] and r["lam_k1_lo"] <= lam[k] <= r["lam_k1_hi"]
    # a closed gap never certifies
    lam = np.array([-1.0, 0.5, 0.5, 1.0])
    assert not setup.shift_bisect(lambda s: setup.inertia(lam, s), 2, -2.0, 2.0, 0.1, 80)["ok"]


QUINTIC = (15.0 / 8.0, -10.0 / 8.0, 3.0 / 8.0)     # (15t - 10t^3 + 3t^5)/8: f(1) = 1, f'(1) = f''(1) = 0


def test_poly_filter_oracle_pins():
    """Generic odd polynomial filters (eq:signpreserving): diagonal H gives the scalar map exactly; any Q gives
    Q diag(phi^m(mu)) Q^T (thm:generic proof P:308-312 holds for every polynomial); the cubic special case is
    the cubic oracle; the quintic sign filter (15t - 10t^3 + 3t^5)/8 preserves signs on [-1, 1] (t phi(t) > 0:
    15 - 10u + 3u^2 has no real root), maps [-1, 1] into itself (phi' = 15(1 - t^2)^2/8 >= 0) and its fixed-depth
    iterate converges to the exact reflector (prop:exact) faster than Newton-Schulz (cubic convergence)."""
    h = np.array([-0.9, -0.2, 0.3, 0.7])
    for coeffs in (QUINTIC, (1.5, -0.5), (1.2, -0.1, 0.05, -0.02)):
        for m in (0, 1, 3):
            X = setup.poly_filter_fixed_depth(np.diag(h), 0.1, 1.0, m, coeffs)
            assert np.max(np.abs(np.diag(X) - setup.poly_filter_scalar(h - 0.1, m, coeffs))) <= 1e-15
    p = workloads.cfg0_controlled(seed=2)
    mu = (p.lam - p.s) / p.alpha
    for coeffs in (QUINTIC, (1.2, -0.1, 0.05, -0.02)):
        for m in (1, 3, 5):
            X = setup.poly_filter_fixed_depth(p.H, p.s, p.alpha, m, coeffs)
            Xcf = closed_form.spectral_matrix(p.Q, setup.poly_filter_scalar(mu, m, coeffs))
            assert np.max(np.abs(X - Xcf)) <= 1e-13
    Xc = setup.poly_filter_fixed_depth(p.H, p.s, p.alpha, 4, (1.5, -0.5))
    assert np.max(np.abs(Xc - setup.filter_fixed_depth(p.H, p.s, p.alpha, 4, 1.5, -0.5))) <= 1e-15
    t = np.linspace(-1, 1, 4001)
    t = t[t != 0]
    f1 = setup.poly_filter_scalar(t, 1, QUINTIC)
    assert np.all(np.sign(f1) == np.sign(t)) and np.all(np.abs(f1) <= 1.0)
    assert np.all(np.diff(f1) >= 0)
    R = closed_form.reflector_explicit_q(p.Q, p.lam, p.s)
    X = setup.poly_filter_fixed_depth(p.H, p.s, p.alpha, 6, QUINTIC)
    assert np.max(np.abs(X - R)) <= 1e-13
    e5 = np.max(np.abs(setup.poly_filter_fixed_depth(p.H, p.s, p.alpha, 4, QUINTIC) - R))
    e3 = np.max(np.abs(setup.poly_filter_fixed_depth(p.H, p.s, p.alpha, 4, (1.5, -0.5)) - R))
    assert e5 < 1e-3 * e3
