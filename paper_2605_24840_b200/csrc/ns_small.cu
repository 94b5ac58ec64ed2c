// Small-d fast path (d <= 96): the whole Newton–Schulz loop of one problem in ONE CTA, with
// X, Y and Z = X Y resident in shared memory (SURVEY §8(a) a9 / K7 for configs[0]-sized problems).
// One launch per call (or per batch: one CTA per problem), no host round trips: the step count is
// decided inside the kernel by the same rule as ns_decide_kernel, so latency is the arithmetic
// (~2 x d^3 FMA per step on one SM's FP64 tensor pipe) instead of 3 launches + a status read per step.
//
// Products use DMMA m8n8k4 fragments read straight from row-major shared memory with a padded pitch
// (d_pad + 4 doubles: the 8 rows of a fragment land 32 B apart, conflict-free per half-warp).  Every
// 8x8 output fragment is computed; the stored matrix takes the upper-triangle value for both (i,j)
// and (j,i), so every iterate is bitwise symmetric, as in the tiled path.
#include <cmath>
#include <cstdint>

#include "ns_internal.h"
#include "ns_ptx.cuh"
#include "ns_small.cuh"

namespace nsr {

template <int DP>
__global__ void __launch_bounds__(kSmallThreads, 1)
    ns_small_kernel(const double* __restrict__ H, long long ldh, long long h_stride, const JobParams* __restrict__ jobs,
                    JobParams job0, LoopParams lp, double* __restrict__ R, long long ldr, long long r_stride,
                    DevState* __restrict__ state) {
  constexpr int P = DP + 4;
  extern __shared__ __align__(16) double sm[];
  double* X = sm;
  double* Y = sm + DP * P;
  double* Z = sm + 2 * DP * P;
  __shared__ double red[kSmallThreads / 32];
  const int job = blockIdx.x;
  const double* Hj = H + (long long)job * h_stride;
  const JobParams jp = jobs ? jobs[job] : job0;   // batch of one: parameters by value (no H2D copy)
  const double s = jp.s, alpha = jp.alpha;
  const int d = lp.d;
  // X_0 = (H - sI)/alpha from the upper triangle, zero padded
  for (int e = threadIdx.x; e < DP * DP; e += kSmallThreads) {
    const int i = e / DP, j = e % DP;
    double v = 0.0;
    if (i < d && j < d) {
      const double h = (i <= j) ? Hj[(long long)i * ldh + j] : Hj[(long long)j * ldh + i];
      v = (i == j) ? (h - s) / alpha : h / alpha;
    }
    X[i * P + j] = v;
  }
  __syncthreads();
  const double sqd = sqrt((double)d);
  int j = 0, flags = 0;
  double r = 0.0, r_prev = 0.0, tr = 0.0;
  while (true) {
    small_product<DP>(X, X, Y);                     // Y_j = X_j^2
    double part = 0.0, tpart = 0.0;
    for (int e = threadIdx.x; e < d * d; e += kSmallThreads) {
      const int i = e / d, c = e % d;
      const double v = Y[i * P + c] - (i == c ? 1.0 : 0.0);
      part += v * v;
    }
    for (int i = threadIdx.x; i < d; i += kSmallThreads) tpart += X[i * P + i];
    r = sqrt(block_sum(part, red));
    tr = block_sum(tpart, red);
    if (!isfinite(r)) {
      flags |= 16;
      break;
    }
    if (j > 0 && r > r_prev * (1.0 + 1e-12) + 1e-10 * sqd) flags |= 8;
    const double rho = lp.tol_mode ? r / sqd : r;
    if (rho < lp.tol) {
      flags |= 1;
      break;
    }
    if (j >= lp.max_steps) {
      flags |= 2;
      break;
    }
    small_product<DP>(X, Y, Z);                     // Z = X_j Y_j
    for (int e = threadIdx.x; e < DP * DP; e += kSmallThreads) {
      const int i = e / DP, c = e % DP;
      X[i * P + c] = fma(lp.cb, Z[i * P + c], lp.ca * X[i * P + c]);
    }
    __syncthreads();
    r_prev = r;
    ++j;
  }
  // R = X_j
  double* Rj = R + (long long)job * r_stride;
  for (int e = threadIdx.x; e < d * d; e += kSmallThreads) {
    const int i = e / d, c = e % d;
    Rj[(long long)i * ldr + c] = X[i * P + c];
  }
  if (threadIdx.x == 0) {
    DevState st{};
    st.j = j;
    st.done = 1;
    st.residual = r;
    st.r_prev = r_prev;
    st.trace = tr;
    st.sw_step = -1;
    const double half = ((double)d - tr) * 0.5;
    long long cert = -1;
    if (!(flags & 16) && isfinite(half)) {
      cert = (long long)floor(fabs(half) + 0.5);
      if (half < 0) cert = -cert;
      if (fabs(half - (double)cert) > 0.25) flags |= 32;
    }
    if (cert != (long long)jp.k) flags |= 4;
    st.cert = cert;
    st.flags = flags;
    state[job] = st;
  }
}

int small_dpad(int d) { return d <= 32 ? 32 : d <= 64 ? 64 : d <= 96 ? 96 : 0; }

cudaError_t launch_small(const double* H, long long ldh, long long h_stride, const JobParams* jobs, JobParams job0,
                         LoopParams lp, double* R, long long ldr, long long r_stride, DevState* state, int batch,
                         cudaStream_t st) {
  static bool attr[3] = {false, false, false};
  const int dp = small_dpad(lp.d);
  const size_t smem = (size_t)3 * dp * (dp + 4) * sizeof(double);
  switch (dp) {
    case 32:
      ns_small_kernel<32><<<batch, kSmallThreads, smem, st>>>(H, ldh, h_stride, jobs, job0, lp, R, ldr, r_stride, state);
      break;
    case 64:
      if (!attr[1]) { cudaFuncSetAttribute(ns_small_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); attr[1] = true; }
      ns_small_kernel<64><<<batch, kSmallThreads, smem, st>>>(H, ldh, h_stride, jobs, job0, lp, R, ldr, r_stride, state);
      break;
    case 96:
      if (!attr[2]) { cudaFuncSetAttribute(ns_small_kernel<96>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); attr[2] = true; }
      ns_small_kernel<96><<<batch, kSmallThreads, smem, st>>>(H, ldh, h_stride, jobs, job0, lp, R, ldr, r_stride, state);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace nsr
