// Algorithm 1 (alg:ssr) on the dense rotated quartic family of §5.3:
// the "step after the path", fused per run into ONE CTA with every matrix in
// shared memory, so a batch of independent runs (k in {1,2,4,8,16} x 32 starts x depths) is one launch.
//
//   E(x) = 1/4 sum y_i^4 + 1/2 sum c_i y_i^2,  y = Q^T x,  c_i = -1 (i <= k), +1 (i > k)
//   g = Q (y^3 + c y),   H = Q diag(mu) Q^T,  mu_i = 3 y_i^2 + c_i
// per outer iteration n (alg:ssr steps 2-8):
//   endpoints lambda_k, lambda_{k+1} = k-th / (k+1)-th smallest mu (exact for this model),
//   shift s by the policy (step 4; DESIGN reading N2b): midpoint (prop:mid), damped midpoint
//   clip(beta s_prev + (1 - beta) mid, [lk + kappa gap, lk1 - kappa gap]), or reuse/refresh (keep s_prev while
//   min(s_prev - lk, lk1 - s_prev) > tau, else the midpoint); stop if the shift's estimated margin <= eps
//   (step 8 "the shift ceases to be admissible", prop:reuse_refresh P:604),
//   alpha = max_i |mu_i - s| = ||H - sI||_2 (divide convention, C1),
//   R~ = phi_m((H - sI)/alpha): m Newton–Schulz steps from X_0 = Q diag((mu - s)/alpha) Q^T
//        (m = 0: the exact reflector Q diag(sgn(mu - s)) Q^T),
//   x_{n+1} = x_n - eta R~ g_n  (eq:discrete_step),  stop when ||g|| <= grad_tol or n = max_iters.
// Success (SPEC's declared criterion): ||g|| <= grad_tol and Morse index of H(x_final) == k.
#include <cmath>
#include <cstdint>

#include "ns_internal.h"
#include "ns_small.cuh"

namespace nsr {

template <int DP>
__global__ void __launch_bounds__(kSmallThreads, 1)
    ns_outer_kernel(const double* __restrict__ Qg, int d, const int* __restrict__ kk, const double* __restrict__ x0,
                    OuterParams p, double* __restrict__ xout, OuterResult* __restrict__ res) {
  constexpr int P = DP + 4;
  extern __shared__ __align__(16) double sm[];
  double* Qs = sm;                 // Q (row-major), padded
  double* A = Qs + DP * P;         // Q diag(.) and then the NS iterate X
  double* Y = A + DP * P;
  double* Z = Y + DP * P;
  double* x = Z + DP * P;          // vectors of length DP
  double* y = x + DP;
  double* g = y + DP;
  double* mu = g + DP;
  double* w = mu + DP;
  __shared__ double red[kSmallThreads / 32];
  __shared__ double sc[4];
  const int run = blockIdx.x;
  const int k = kk[run];
  for (int e = threadIdx.x; e < DP * DP; e += kSmallThreads) {
    const int i = e / DP, j = e % DP;
    Qs[i * P + j] = (i < d && j < d) ? Qg[(long long)i * d + j] : 0.0;
  }
  for (int i = threadIdx.x; i < DP; i += kSmallThreads) x[i] = (i < d) ? x0[(long long)run * d + i] : 0.0;
  __syncthreads();
  int n = 0, refreshes = 0, stop = 0;
  double gn = 0.0;
  double s_prev = __longlong_as_double(0x7ff8000000000000ll);   // NaN: no shift yet
  while (true) {
    // y = Q^T x ; mu ; g = Q (y^3 + c y)
    for (int i = threadIdx.x; i < DP; i += kSmallThreads) {
      double a = 0.0;
      for (int j = 0; j < d; ++j) a = fma(Qs[j * P + i], x[j], a);
      y[i] = a;
      const double c = (i < k) ? -1.0 : 1.0;
      mu[i] = (i < d) ? 3.0 * a * a + c : 0.0;
      w[i] = (i < d) ? a * a * a + c * a : 0.0;
    }
    __syncthreads();
    double gp = 0.0;
    for (int i = threadIdx.x; i < DP; i += kSmallThreads) {
      double a = 0.0;
      for (int j = 0; j < d; ++j) a = fma(Qs[i * P + j], w[j], a);
      g[i] = a;
      gp += a * a;
    }
    gn = sqrt(block_sum(gp, red));
    if (!(gn > p.grad_tol)) { stop = 0; break; }   // also stops on NaN
    if (n >= p.max_iters) { stop = 1; break; }
    // endpoints: k-th and (k+1)-th smallest mu (rank by counting, ties by index)
    for (int i = threadIdx.x; i < d; i += kSmallThreads) {
      int rank = 0;
      for (int j = 0; j < d; ++j) rank += (mu[j] < mu[i]) || (mu[j] == mu[i] && j < i);
      if (rank == k - 1) sc[0] = mu[i];
      if (rank == k) sc[1] = mu[i];
    }
    __syncthreads();
    // step 4: every thread takes the same decision from the same shared endpoints
    const double lk = sc[0], lk1 = sc[1];
    const double mid = 0.5 * (lk + lk1);
    double s = mid;
    bool fresh = true;
    if (n > 0 && p.policy == 1) {
      const double gap = lk1 - lk;
      const double blend = __dadd_rn(__dmul_rn(p.damp, s_prev), __dmul_rn(1.0 - p.damp, mid));
      s = fmin(fmax(blend, __dadd_rn(lk, __dmul_rn(p.clip, gap))), __dsub_rn(lk1, __dmul_rn(p.clip, gap)));
      fresh = false;
    } else if (n > 0 && p.policy == 2) {
      if (fmin(s_prev - lk, lk1 - s_prev) > p.reuse_margin) {
        s = s_prev;
        fresh = false;
      }
    }
    if (!(fmin(s - lk, lk1 - s) > p.eps)) { stop = 2; break; }   // inadmissible shift: no update
    refreshes += fresh ? 1 : 0;
    s_prev = s;
    double am = 0.0;
    for (int i = threadIdx.x; i < d; i += kSmallThreads) am = fmax(am, fabs(mu[i] - s));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) am = fmax(am, __shfl_xor_sync(0xffffffffu, am, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = am;
    __syncthreads();
    double alpha = 0.0;
    for (int ww = 0; ww < kSmallThreads / 32; ++ww) alpha = fmax(alpha, red[ww]);
    __syncthreads();
    // X_0 = Q diag(f(mu)) Q^T with f = (mu - s)/alpha, or sgn(mu - s) for the exact reflector
    for (int e = threadIdx.x; e < DP * DP; e += kSmallThreads) {
      const int i = e / DP, j = e % DP;
      double f = 0.0;
      if (j < d) f = (p.m == 0) ? (mu[j] > s ? 1.0 : (mu[j] < s ? -1.0 : 0.0)) : (mu[j] - s) / alpha;
      Z[i * P + j] = Qs[i * P + j] * f;
    }
    __syncthreads();
    small_product<DP>(Z, Qs, A);
    for (int step = 0; step < p.m; ++step) {
      small_product<DP>(A, A, Y);
      small_product<DP>(A, Y, Z);
      for (int e = threadIdx.x; e < DP * DP; e += kSmallThreads) {
        const int i = e / DP, j = e % DP;
        A[i * P + j] = fma(-0.5, Z[i * P + j], 1.5 * A[i * P + j]);
      }
      __syncthreads();
    }
    // x <- x - eta R~ g
    for (int i = threadIdx.x; i < DP; i += kSmallThreads) {
      double a = 0.0;
      for (int j = 0; j < d; ++j) a = fma(A[i * P + j], g[j], a);
      w[i] = a;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < d; i += kSmallThreads) x[i] = fma(-p.eta, w[i], x[i]);
    __syncthreads();
    ++n;
  }
  // Morse index of H(x_final) = #{mu_i < 0}
  int neg = 0;
  for (int i = 0; i < d; ++i) neg += (mu[i] < 0.0);
  for (int i = threadIdx.x; i < d; i += kSmallThreads) xout[(long long)run * d + i] = x[i];
  if (threadIdx.x == 0) {
    OuterResult r;
    r.iters = n;
    r.morse_index = neg;
    r.grad_norm = gn;
    r.success = (gn <= p.grad_tol && neg == k) ? 1 : 0;
    r.stop_reason = stop;
    r.refreshes = refreshes;
    r.pad = 0;
    r.s_last = s_prev;
    res[run] = r;
  }
}

cudaError_t launch_outer(const double* Q, int d, const int* k, const double* x0, OuterParams p, double* xout,
                         OuterResult* res, int nruns, cudaStream_t st) {
  const int dp = small_dpad(d);
  const size_t smem = ((size_t)4 * dp * (dp + 4) + 5 * (size_t)dp) * sizeof(double);
  switch (dp) {
    case 32:
      ns_outer_kernel<32><<<nruns, kSmallThreads, smem, st>>>(Q, d, k, x0, p, xout, res);
      break;
    case 64:
      cudaFuncSetAttribute(ns_outer_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      ns_outer_kernel<64><<<nruns, kSmallThreads, smem, st>>>(Q, d, k, x0, p, xout, res);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace nsr
