// Shift/scale setup on the device ("the step before the path").
//
// alg:ssr step 5 and the recommended default realization: choose alpha so
// that the spectrum of (H - sI)/alpha lies in [-1, 1]; when no spectral-norm estimate is available
// use the cheaper surrogate ||H - sI||_inf (disc "scaling choice"), which for symmetric H
// is the Gershgorin bound max_i (|H_ii - s| + sum_{j != i} |H_ij|) >= ||H - sI||_2.
// Only the upper triangle of H is read: row i's sum is its upper part (j >= i, coalesced) plus the
// strict upper part of column i (rows j < i, coalesced across a warp's 32 consecutive columns).
#include <cmath>
#include <cstdint>

#include "ns_internal.h"

namespace nsr {

// part[i] = sum_{j >= i} |H_ij - s delta_ij|   (one warp per row)
__global__ void __launch_bounds__(256) ns_rowsum_upper_kernel(const double* __restrict__ H, long long ldh, int d,
                                                              double s, double* __restrict__ part) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= d) return;
  const int i = warp;
  double acc = 0.0;
  for (int j = i + lane; j < d; j += 32) {
    const double h = H[(long long)i * ldh + j];
    acc += fabs(j == i ? h - s : h);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) part[i] = acc;
}

// part[j] += sum_{i < j} |H_ij|   (column j of the strict upper triangle = row j of the strict lower)
__global__ void __launch_bounds__(256) ns_colsum_upper_kernel(const double* __restrict__ H, long long ldh, int d,
                                                              double* __restrict__ part) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  double acc = 0.0;
  for (int i = 0; i < j; ++i) acc += fabs(H[(long long)i * ldh + j]);
  part[j] += acc;
}

// max that propagates NaN (fmax drops a NaN operand, which would turn a NaN row sum into a finite,
// wrong bound: the Gershgorin guarantee alpha >= ||H - sI||_2 must not silently fail)
__device__ __forceinline__ double nan_max(double a, double b) { return (a != a || b != b) ? (a + b) : fmax(a, b); }

__global__ void __launch_bounds__(256) ns_max_kernel(const double* __restrict__ v, int n, double* out) {
  __shared__ double red[8];
  double m = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) m = nan_max(m, v[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = nan_max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t = nan_max(t, red[w]);
    out[0] = t;
  }
}

cudaError_t launch_scale_bound(const double* H, long long ldh, int d, double s, double* part, double* out,
                               cudaStream_t st) {
  ns_rowsum_upper_kernel<<<(d * 32 + 255) / 256, 256, 0, st>>>(H, ldh, d, s, part);
  ns_colsum_upper_kernel<<<(d + 255) / 256, 256, 0, st>>>(H, ldh, d, part);
  ns_max_kernel<<<1, 256, 0, st>>>(part, d, out);
  return cudaGetLastError();
}

}  // namespace nsr
