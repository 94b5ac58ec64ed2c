"""Input recipes for BASELINE.json configs[0..4] (readings C10-C14 in DESIGN.md §Inputs).

All randomness: numpy ``Generator(PCG64(seed))``; cfg1 uses one spawned stream per
matrix (``SeedSequence(seed).spawn(2048)``).  Every H is symmetrised
``H <- (H + H^T)/2`` before use, so reading the upper triangle (CUDA path) and
reading all of H (oracle) see the same matrix.  This module contains no
Newton–Schulz arithmetic.
"""
import math
from dataclasses import dataclass, field

import numpy as np


def _rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def haar_q(rng, d):
    """Haar orthogonal Q: QR of a seeded N(0,1) matrix, sign-fixed by diag(R) (BASELINE cfg0/cfg1)."""
    G = rng.standard_normal((d, d))
    Q, Rr = np.linalg.qr(G)
    return Q * np.sign(np.diag(Rr))[None, :]


def _sym(H):
    return 0.5 * (H + H.T)


@dataclass
class Problem:
    """One NS reflector problem.  lam/Q/Vh are the generator's ground truth (None if unknown)."""
    name: str
    d: int
    k: int
    s: float
    alpha: float
    max_steps: int
    tol: float
    tol_mode: int            # 0 = ||X^2-I||_F < tol ; 1 = ||X^2-I||_F/sqrt(d) < tol
    H: np.ndarray = None     # d x d float64 (None when formed on device)
    lam: np.ndarray = None   # eigenvalues in generator order (unsorted)
    Q: np.ndarray = None     # explicit orthogonal factor (Haar)
    Vh: np.ndarray = None    # Householder vectors (n x d), Q = H_1 ... H_n
    extra: dict = field(default_factory=dict)


# --------------------------------------------------------------------------- cfg0
def cfg0_controlled(seed=0, d=64, k=3):
    """configs[0]: d=64, k=3, Haar Q; lambda_1..3 ~ U[-2,-0.5], rest ~ U[0.5,2];
    s = midpoint (lambda_(3)+lambda_(4))/2; alpha = max(|lambda_(1)-s|, |lambda_(d)-s|);
    tol 1e-12 absolute, 100 steps.  Draw order: lambda_neg, lambda_pos, G (C10)."""
    rng = _rng(seed)
    lam_neg = rng.uniform(-2.0, -0.5, k)
    lam_pos = rng.uniform(0.5, 2.0, d - k)
    Q = haar_q(rng, d)
    lam = np.concatenate([lam_neg, lam_pos])
    H = _sym((Q * lam[None, :]) @ Q.T)
    ls = np.sort(lam)
    s = 0.5 * (ls[k - 1] + ls[k])
    alpha = max(abs(ls[0] - s), abs(ls[-1] - s))
    return Problem("cfg0", d, k, s, alpha, 100, 1e-12, 0, H=H, lam=lam, Q=Q)


# --------------------------------------------------------------------------- cfg1
def cfg1_batched(seed=0, n_matrices=2048, d=256, first=0, count=None):
    """configs[1]: 2048 Haar matrices of d=256, k ~ U{1..32}, g = 10^U(-3,-1),
    lambda_1..k ~ U[-1,-g/2], rest ~ U[g/2,1]; shifts mid, mid+0.4 gap, mid-0.4 gap
    (gap = realised lambda_(k+1)-lambda_(k)), alpha = 1+|s|; tol 1e-12 abs, 100 steps (C11).
    Per-matrix stream: SeedSequence(seed).spawn(n)[b]; draw order k, g, lambda_neg,
    lambda_pos, G, v (unit direction probe).  Returns a list of Problems, one per
    (matrix, shift), matrix-major: [b0 mid, b0 +, b0 -, b1 mid, ...]."""
    count = n_matrices - first if count is None else count
    streams = np.random.SeedSequence(seed).spawn(n_matrices)
    out = []
    for b in range(first, first + count):
        rng = np.random.Generator(np.random.PCG64(streams[b]))
        k = int(rng.integers(1, 33))
        g = 10.0 ** rng.uniform(-3.0, -1.0)
        lam_neg = rng.uniform(-1.0, -g / 2.0, k)
        lam_pos = rng.uniform(g / 2.0, 1.0, d - k)
        Q = haar_q(rng, d)
        v = rng.standard_normal(d)
        v /= np.linalg.norm(v)
        lam = np.concatenate([lam_neg, lam_pos])
        H = _sym((Q * lam[None, :]) @ Q.T)
        ls = np.sort(lam)
        gap = ls[k] - ls[k - 1]
        mid = 0.5 * (ls[k - 1] + ls[k])
        for tag, s in (("mid", mid), ("plus", mid + 0.4 * gap), ("minus", mid - 0.4 * gap)):
            out.append(Problem(f"cfg1[{b}].{tag}", d, k, s, 1.0 + abs(s), 100, 1e-12, 0, H=H, lam=lam,
                               Q=Q, extra=dict(matrix=b, shift=tag, gap=gap, g=g, probe=v)))
    return out


# --------------------------------------------------------------------------- cfg2
def allen_cahn_field(seed, n=64, modes=8, kmax=4):
    """Smooth periodic field u on the n x n grid x_i = i/n (reading C12):
    u = sum_m a_m cos(2 pi (kx x + ky y) + phi_m), (kx,ky) uniform on {-4..4}^2 \\ {(0,0)}
    (rejection), a_m ~ N(0,1)/(1+kx^2+ky^2), phi_m ~ U[0, 2pi); draw order per mode:
    (kx,ky), a, phi.  Normalised to max|u| = 1.  Flattened with p = iy*n + ix."""
    rng = _rng(seed)
    x = np.arange(n) / n
    X, Y = np.meshgrid(x, x, indexing="xy")     # X[iy, ix] = x_ix, Y[iy, ix] = y_iy
    u = np.zeros((n, n))
    for _ in range(modes):
        while True:
            kx, ky = (int(t) for t in rng.integers(-kmax, kmax + 1, size=2))
            if (kx, ky) != (0, 0):
                break
        a = rng.standard_normal() / (1.0 + kx * kx + ky * ky)
        phi = rng.uniform(0.0, 2.0 * math.pi)
        u += a * np.cos(2.0 * math.pi * (kx * X + ky * Y) + phi)
    u /= np.max(np.abs(u))
    return u.reshape(-1)


def allen_cahn_hessian(u, n=64, eps=0.04):
    """H = eps^2 L_h + diag(3u^2 - 1), L_h the periodic 5-point negative Laplacian / h^2,
    h = 1/n, index p = iy*n + ix (configs[2]; C12)."""
    h = 1.0 / n
    d = n * n
    H = np.zeros((d, d))
    c = eps * eps / (h * h)
    for iy in range(n):
        for ix in range(n):
            p = iy * n + ix
            H[p, p] += 4.0 * c
            for jx, jy in ((ix + 1, iy), (ix - 1, iy), (ix, iy + 1), (ix, iy - 1)):
                q = (jy % n) * n + (jx % n)
                H[p, q] -= c
    H[np.arange(d), np.arange(d)] += 3.0 * np.asarray(u) ** 2 - 1.0
    return _sym(H)


def gershgorin_alpha(H, s):
    """alpha = max_i (|H_ii - s| + sum_{j != i} |H_ij|)  (configs[2] "alpha from the Gershgorin bound")."""
    diag = np.diag(H)
    off = np.sum(np.abs(H), axis=1) - np.abs(diag)
    return float(np.max(np.abs(diag - s) + off))


def cfg2_allen_cahn(seed=0, s=None, u=None, n=64, eps=0.04, k=5):
    """configs[2]: Allen–Cahn Hessian, d = 4096, k = 5.  s must be supplied by the
    oracle (midpoint of its Jacobi lambda_5, lambda_6; tests/golden/cfg2_*.json);
    alpha = Gershgorin at that s; tol 1e-12 abs, 100 steps (C12).  u overrides the
    seeded field (u = 0 gives the closed-form DFT case)."""
    u = allen_cahn_field(seed, n=n) if u is None else np.asarray(u, dtype=np.float64)
    H = allen_cahn_hessian(u, n=n, eps=eps)
    alpha = gershgorin_alpha(H, s) if s is not None else None
    return Problem(f"cfg2[seed={seed}]", n * n, k, s, alpha, 100, 1e-12, 0, H=H, extra=dict(u=u))


# --------------------------------------------------------------------------- cfg3 / cfg4
def householder_spectrum(seed, d, k, margin, n_house):
    """lambda_1..k ~ U[-1,-margin], rest ~ U[margin,1] (negatives first, unsorted), then the
    n_house Householder vectors v_i ~ N(0,1)^d (reading C13)."""
    rng = _rng(seed)
    lam = np.concatenate([rng.uniform(-1.0, -margin, k), rng.uniform(margin, 1.0, d - k)])
    Vh = rng.standard_normal((n_house, d))
    return lam, Vh


def householder_form_numpy(Vh, lam):
    """H = Q diag(lam) Q^T with Q = H_1...H_n, formed inside-out M <- H_i M H_i, i = n..1.
    Each step is the symmetric rank-2 update M + v a^T + a v^T with w = M v,
    beta = 2/(v^T v), a = -beta w + (beta^2/2)(v^T w) v."""
    M = np.diag(np.asarray(lam, dtype=np.float64))
    for i in range(Vh.shape[0] - 1, -1, -1):
        v = Vh[i]
        beta = 2.0 / float(v @ v)
        w = M @ v
        a = -beta * w + 0.5 * beta * beta * float(v @ w) * v
        M += np.outer(v, a)
        M += np.outer(a, v)
    return _sym(M)


def householder_form_torch(Vh, lam, device):
    """Same recipe as householder_form_numpy, evaluated with torch on `device` (input
    preparation only; used by bench/tests to build d >= 16384 inputs in HBM)."""
    import torch
    M = torch.diag(torch.as_tensor(np.asarray(lam), dtype=torch.float64, device=device))
    V = torch.as_tensor(Vh, dtype=torch.float64, device=device)
    for i in range(V.shape[0] - 1, -1, -1):
        v = V[i]
        beta = 2.0 / float(v @ v)
        w = M @ v
        a = -beta * w + 0.5 * beta * beta * float(v @ w) * v
        M.addr_(v, a)
        M.addr_(a, v)
    M.add_(M.T.clone()).mul_(0.5)
    return M


def householder_form_fast(Vh, lam, device=None):
    """Same H = Q diag(lam) Q^T (Q = H_1...H_n), formed through the compact WY
    representation Q = I - V T V^T (V = [v_1..v_n], T upper triangular with
    T_ii = beta_i = 2/(v_i^T v_i), T[:i, i] = -beta_i T[:i,:i] V[:, :i]^T v_i):
        H = Lambda + W A^T + A W^T,  A = V T,  U = Lambda V,  M = U^T V,  W = A M / 2 - U.
    Two rank-n GEMMs instead of n rank-2 sweeps, so d = 16384..49152 inputs form in
    seconds.  numpy on the host (device=None) or torch on `device`.  Exactly symmetric."""
    Vh = np.asarray(Vh, dtype=np.float64)
    lam = np.asarray(lam, dtype=np.float64)
    n = Vh.shape[0]
    V = Vh.T                                   # d x n, columns v_i
    G = Vh @ V                                 # n x n Gram matrix v_i^T v_j
    T = np.zeros((n, n))
    for i in range(n):
        beta = 2.0 / G[i, i]
        T[i, i] = beta
        if i:
            T[:i, i] = -beta * (T[:i, :i] @ G[:i, i])
    if device is None:
        A = V @ T
        U = lam[:, None] * V
        M = U.T @ V
        W = 0.5 * (A @ M) - U
        Gm = W @ A.T
        H = Gm + Gm.T
        H[np.diag_indices_from(H)] += lam
        return H
    import torch
    Vt = torch.as_tensor(np.ascontiguousarray(V), dtype=torch.float64, device=device)
    Tt = torch.as_tensor(T, dtype=torch.float64, device=device)
    lt = torch.as_tensor(lam, dtype=torch.float64, device=device)
    A = Vt @ Tt
    U = lt[:, None] * Vt
    M = U.T @ Vt
    W = 0.5 * (A @ M) - U
    H = W @ A.T
    H = H + H.T
    H.diagonal().add_(lt)
    return H


def cfg3_dense(seed=1, d=16384, k=1024, margin=0.05, n_house=64, form=True, mode="tol"):
    """configs[3]: d=16384, k=1024, Q = 64 Householders, s = 0, alpha = 1.05.
    mode "tol": ||X^2-I||_F/sqrt(d) < 1e-10 (C3), max 100 steps; mode "fixed30": tol 0,
    30 steps (C5).  `d`/`k` may be reduced with k = d/16 for CPU-sized cases."""
    lam, Vh = householder_spectrum(seed, d, k, margin, n_house)
    H = householder_form_numpy(Vh, lam) if form else None
    if mode == "fixed30":
        tol, max_steps = 0.0, 30
    else:
        tol, max_steps = 1e-10, 100
    return Problem(f"cfg3[d={d},{mode}]", d, k, 0.0, 1.05, max_steps, tol, 1, H=H, lam=lam, Vh=Vh)


def cfg4_sharded(seed=1, d=49152, k=4096, margin=0.02, n_house=32, form=True):
    """configs[4]: d=49152, k=4096, 32 Householders, s=0, alpha=1.05, /sqrt(d) tol 1e-10.
    The oracle sub-problem is the same recipe at d=4096, k=round(4096*4096/49152)=341 (C14)."""
    lam, Vh = householder_spectrum(seed, d, k, margin, n_house)
    H = householder_form_numpy(Vh, lam) if form else None
    return Problem(f"cfg4[d={d}]", d, k, 0.0, 1.05, 100, 1e-10, 1, H=H, lam=lam, Vh=Vh)


# --------------------------------------------------------------------------- N2: target-index scan
def rotated_quartic_scan(seed=0, d=64, ks=(1, 2, 4, 8, 16), n_starts=32, radius=4.0):
    """§5.3 target-index scan inputs: one Haar Q (shared), and n_starts matched random starts
    x0 ~ radius * N(0, I)/sqrt(d) (the same starts for every k, "matched random starts").
    The paper does not state the start distribution or the c_i magnitudes; unit |c_i| and
    this start recipe are DESIGN.md readings."""
    rng = _rng(seed)
    Q = haar_q(rng, d)
    starts = radius * rng.standard_normal((n_starts, d)) / math.sqrt(d)
    return Q, list(ks), starts
