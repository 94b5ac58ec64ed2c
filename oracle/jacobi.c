/* Cyclic Jacobi eigendecomposition of a dense real symmetric matrix.
 *
 * TEST INFRASTRUCTURE ONLY (oracle/).  Shares no code with the CUDA path.
 *
 * "Eigensolver: cyclic Jacobi rotations, convergence when off-diagonal
 * Frobenius norm <= 1e-13 * ||A||_F, sweep cap 60".  The cyclic ordering used
 * is the round-robin ("tournament") ordering: a sweep is n-1 rounds, each round
 * annihilates n/2 disjoint (p,q) pairs, so every off-diagonal pair is visited
 * once per sweep, as in any cyclic Jacobi.  Disjoint pairs commute, which lets
 * a round be applied as  A <- J^T A J  by one pass over rows (rows p,q of every
 * pair) and one pass over columns (done row by row), and  V <- V J.
 *
 * Rotation (Golub & Van Loan, symmetric Schur 2x2): with
 *   theta = (a_qq - a_pp) / (2 a_pq),  t = sgn(theta)/(|theta| + sqrt(theta^2+1)),
 *   c = 1/sqrt(1+t^2),  s = t c,
 * J = [[c, s], [-s, c]] on coordinates (p,q) makes (J^T A J)_pq = 0.
 *
 * Output: eigenvalues ascending in w[0..d-1]; V row-major d x d whose COLUMNS
 * are the matching orthonormal eigenvectors (H = V diag(w) V^T).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

static void round_pairs(int n, int r, int* P, int* Q) {
  /* circle method on n (even) players: player n-1 fixed, others rotate by r */
  int m = n - 1;
  P[0] = r % m;
  Q[0] = m;
  for (int i = 1; i < n / 2; ++i) {
    P[i] = (r + i) % m;
    Q[i] = (r - i + m) % m;
  }
  for (int i = 0; i < n / 2; ++i)
    if (P[i] > Q[i]) { int t = P[i]; P[i] = Q[i]; Q[i] = t; }
}

static double offdiag_norm(int d, const double* A) {
  double s = 0.0;
#pragma omp parallel for reduction(+ : s) schedule(static)
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j)
      if (i != j) s += A[(size_t)i * d + j] * A[(size_t)i * d + j];
  return sqrt(s);
}

static double frob_norm(int d, const double* A) {
  double s = 0.0;
#pragma omp parallel for reduction(+ : s) schedule(static)
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) s += A[(size_t)i * d + j] * A[(size_t)i * d + j];
  return sqrt(s);
}

/* Returns number of sweeps performed (>=0), or -1 if not converged within max_sweeps. */
int jacobi_eigh(int d, double* A, double* V, double* w, double rel_tol, int max_sweeps) {
  int n = d + (d & 1);
  int* P = (int*)malloc(sizeof(int) * (n / 2));
  int* Q = (int*)malloc(sizeof(int) * (n / 2));
  double* C = (double*)malloc(sizeof(double) * (n / 2));
  double* S = (double*)malloc(sizeof(double) * (n / 2));
  int* part = (int*)malloc(sizeof(int) * n); /* partner index and role per coordinate */
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) V[(size_t)i * d + j] = (i == j) ? 1.0 : 0.0;
  double target = rel_tol * frob_norm(d, A);
  int sweep = 0, converged = 0;
  if (offdiag_norm(d, A) <= target) converged = 1;
  while (!converged && sweep < max_sweeps) {
    for (int r = 0; r < n - 1; ++r) {
      round_pairs(n, r, P, Q);
      int np = 0;
      /* 1. rotations of this round, from the current 2x2 blocks */
      for (int i = 0; i < n / 2; ++i) {
        int p = P[i], q = Q[i];
        if (q >= d) continue; /* padding player */
        double apq = A[(size_t)p * d + q];
        if (apq == 0.0) continue;
        double app = A[(size_t)p * d + p], aqq = A[(size_t)q * d + q];
        double theta = (aqq - app) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(1.0 + t * t);
        P[np] = p; Q[np] = q; C[np] = c; S[np] = t * c; ++np;
      }
      if (np == 0) continue;
      /* 2. rows: A <- J^T A  (rows p, q of each pair) */
#pragma omp parallel for schedule(static)
      for (int i = 0; i < np; ++i) {
        double* rp = A + (size_t)P[i] * d;
        double* rq = A + (size_t)Q[i] * d;
        double c = C[i], s = S[i];
        for (int j = 0; j < d; ++j) {
          double x = rp[j], y = rq[j];
          rp[j] = c * x - s * y;
          rq[j] = s * x + c * y;
        }
      }
      /* 3. columns: A <- A J and V <- V J, row by row */
#pragma omp parallel for schedule(static)
      for (int row = 0; row < d; ++row) {
        double* a = A + (size_t)row * d;
        double* v = V + (size_t)row * d;
        for (int i = 0; i < np; ++i) {
          int p = P[i], q = Q[i];
          double c = C[i], s = S[i];
          double x = a[p], y = a[q];
          a[p] = c * x - s * y;
          a[q] = s * x + c * y;
          x = v[p]; y = v[q];
          v[p] = c * x - s * y;
          v[q] = s * x + c * y;
        }
      }
      /* the rotation annihilates a_pq exactly in exact arithmetic */
      for (int i = 0; i < np; ++i) {
        A[(size_t)P[i] * d + Q[i]] = 0.0;
        A[(size_t)Q[i] * d + P[i]] = 0.0;
      }
    }
    ++sweep;
    if (offdiag_norm(d, A) <= target) converged = 1;
  }
  /* eigenvalues = diagonal; sort ascending (insertion sort on an index array) */
  int* idx = part;
  for (int i = 0; i < d; ++i) { idx[i] = i; w[i] = A[(size_t)i * d + i]; }
  for (int i = 1; i < d; ++i) {
    int k = idx[i], j = i - 1;
    while (j >= 0 && w[idx[j]] > w[k]) { idx[j + 1] = idx[j]; --j; }
    idx[j + 1] = k;
  }
  double* wtmp = (double*)malloc(sizeof(double) * d);
  double* rowtmp = (double*)malloc(sizeof(double) * d);
  for (int i = 0; i < d; ++i) wtmp[i] = w[idx[i]];
  memcpy(w, wtmp, sizeof(double) * d);
  for (int row = 0; row < d; ++row) {
    double* v = V + (size_t)row * d;
    for (int i = 0; i < d; ++i) rowtmp[i] = v[idx[i]];
    memcpy(v, rowtmp, sizeof(double) * d);
  }
  free(wtmp); free(rowtmp);
  free(P); free(Q); free(C); free(S); free(part);
  return converged ? sweep : -1;
}
