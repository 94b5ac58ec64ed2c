"""Algorithm 1 on the dense rotated quartic (oracle; test infrastructure).

alg:ssr steps 2-8, in the paper's order, on E(x) = 1/4 sum y^4 + 1/2 sum c y^2,
y = Q^T x, c_i = -1 (i <= k), +1 (i > k) (§5.3):
    g = Q (y^3 + c y),  H = Q diag(mu) Q^T with mu = 3 y^2 + c             (step 2)
    lambda_k, lambda_{k+1} = k-th and (k+1)-th smallest mu                 (step 3, exact endpoints)
    s = (lambda_k + lambda_{k+1}) / 2                                      (step 4, midpoint, prop:mid)
    alpha = ||H - sI||_2 = max_i |mu_i - s|                                (step 5, divide convention C1)
    R~ = m Newton-Schulz steps from X_0 = (H - sI)/alpha, or sgn(H - sI)   (step 6)
    x <- x - eta R~ g                                                      (step 7, eq:discrete_step)
    stop when ||g|| <= grad_tol or the iteration budget is spent           (step 8)
Success (SPEC's declared criterion): ||g|| <= grad_tol and Morse index of H(x_final) == k.
"""
import numpy as np


def gradient_and_mu(Q, k, x):
    d = Q.shape[0]
    c = np.where(np.arange(d) < k, -1.0, 1.0)
    y = Q.T @ x
    return Q @ (y ** 3 + c * y), 3.0 * y * y + c


def run(Q, k, x0, m, eta, max_iters, grad_tol):
    Q = np.asarray(Q, dtype=np.float64)
    x = np.array(x0, dtype=np.float64, copy=True)
    n = 0
    while True:
        g, mu = gradient_and_mu(Q, k, x)
        gn = float(np.linalg.norm(g))
        if not (gn > grad_tol) or n >= max_iters:
            break
        srt = np.sort(mu)
        s = 0.5 * (srt[k - 1] + srt[k])
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
    return dict(x=x, iters=n, grad_norm=gn, morse_index=morse, success=bool(gn <= grad_tol and morse == k))
