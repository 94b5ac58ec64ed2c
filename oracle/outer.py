"""Algorithm 1 on the dense rotated quartic (oracle; test infrastructure).

alg:ssr steps 2-8, in the paper's order, on E(x) = 1/4 sum y^4 + 1/2 sum c y^2,
y = Q^T x, c_i = -1 (i <= k), +1 (i > k) (§5.3):
    g = Q (y^3 + c y),  H = Q diag(mu) Q^T with mu = 3 y^2 + c             (step 2)
    stop when ||g|| <= grad_tol or the iteration budget is spent           (step 8, tested before the update)
    lambda_k, lambda_{k+1} = k-th and (k+1)-th smallest mu                 (step 3, exact endpoints)
    s_n by the shift policy                                                (step 4):
        midpoint        s = (lambda_k + lambda_{k+1}) / 2                  (prop:mid)
        damped          s = clip(beta s_{n-1} + (1 - beta) mid, [lambda_k + kappa gap, lambda_{k+1} - kappa gap])
                        ("blend the previous admissible shift with the new midpoint and clip back into the
                        estimated gap"; DESIGN reading C24: beta = damp, kappa = clip in (0, 1/2]); n = 0: mid
        reuse_refresh   keep s_{n-1} while its estimated margin min(s - lambda_k, lambda_{k+1} - s) > tau
                        (tau = reuse_margin), otherwise s = mid                    (C25; n = 0: mid)
    stop when the chosen shift is not admissible: estimated margin <= eps   (step 8, prop:reuse_refresh
                        P:604: "If m_hat > eps, then s is admissible"; eps = endpoint error bound, 0 here
                        since the model's endpoints are exact -- C26)
    alpha = ||H - sI||_2 = max_i |mu_i - s|                                (step 5, divide convention C1)
    R~ = m Newton-Schulz steps from X_0 = (H - sI)/alpha, or sgn(H - sI)   (step 6)
    x <- x - eta R~ g                                                      (step 7, eq:discrete_step)
Success (SPEC's declared criterion): ||g|| <= grad_tol and Morse index of H(x_final) == k.
"""
import numpy as np

POLICIES = ("midpoint", "damped", "reuse_refresh")
STOP_GRAD, STOP_BUDGET, STOP_INADMISSIBLE = 0, 1, 2


def gradient_and_mu(Q, k, x):
    d = Q.shape[0]
    c = np.where(np.arange(d) < k, -1.0, 1.0)
    y = Q.T @ x
    return Q @ (y ** 3 + c * y), 3.0 * y * y + c


def choose_shift(policy, lam_k, lam_k1, s_prev, damp=0.5, clip=0.25, reuse_margin=0.0):
    """alg:ssr step 4.  Returns (s, refreshed): refreshed = the fresh midpoint was taken."""
    mid = 0.5 * (lam_k + lam_k1)
    if policy == "midpoint" or s_prev is None:
        return mid, True
    if policy == "damped":
        gap = lam_k1 - lam_k
        s = damp * s_prev + (1.0 - damp) * mid
        lo, hi = lam_k + clip * gap, lam_k1 - clip * gap
        return min(max(s, lo), hi), False
    if policy == "reuse_refresh":
        margin = min(s_prev - lam_k, lam_k1 - s_prev)
        if margin > reuse_margin:
            return s_prev, False
        return mid, True
    raise ValueError(policy)


def run(Q, k, x0, m, eta, max_iters, grad_tol, policy="midpoint", damp=0.5, clip=0.25, reuse_margin=0.0,
        eps=0.0):
    if policy not in POLICIES:
        raise ValueError(policy)
    Q = np.asarray(Q, dtype=np.float64)
    x = np.array(x0, dtype=np.float64, copy=True)
    n = 0
    s_prev = None
    shifts, refreshes = [], 0
    while True:
        g, mu = gradient_and_mu(Q, k, x)
        gn = float(np.linalg.norm(g))
        if not (gn > grad_tol):
            stop = STOP_GRAD
            break
        if n >= max_iters:
            stop = STOP_BUDGET
            break
        srt = np.sort(mu)
        lam_k, lam_k1 = srt[k - 1], srt[k]
        s, fresh = choose_shift(policy, lam_k, lam_k1, s_prev, damp, clip, reuse_margin)
        if not (min(s - lam_k, lam_k1 - s) > eps):
            stop = STOP_INADMISSIBLE
            break
        refreshes += int(fresh)
        shifts.append(s)
        s_prev = s
        alpha = float(np.max(np.abs(mu - s)))
        if m == 0:
            R = (Q * np.sign(mu - s)) @ Q.T
        else:
            X = (Q * ((mu - s) / alpha)) @ Q.T
            for _ in range(m):
                X = 1.5 * X - 0.5 * (X @ (X @ X))
                X = 0.5 * (X + X.T)
            R = X
        x = x - eta * (R @ g)
        n += 1
    morse = int(np.sum(mu < 0.0))
    return dict(x=x, iters=n, grad_norm=gn, morse_index=morse, success=bool(gn <= grad_tol and morse == k),
                stop_reason=stop, refreshes=refreshes, shifts=shifts)
