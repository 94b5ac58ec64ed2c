// Shared-memory-resident FP64 DMMA helpers for one CTA (d_pad <= 96): used by the fused small-d
// Newton–Schulz kernel (ns_small.cu) and the fused Algorithm-1 outer loop (ns_outer.cu).
#pragma once
#include <cmath>
#include <cstdint>

#include "ns_internal.h"
#include "ns_ptx.cuh"

namespace nsr {

constexpr int kSmallThreads = 256;

template <int DP>
__device__ __forceinline__ void small_product(const double* __restrict__ A, const double* __restrict__ B,
                                              double* __restrict__ C) {
  // C[i][j] = sum_k A[i][k] B[j][k]   (both operands row panels of symmetric matrices)
  constexpr int P = DP + 4;
  constexpr int NF = DP / 8;               // fragments per dimension
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  for (int f = warp; f < NF * NF; f += kSmallThreads / 32) {
    const int fi = f / NF, fj = f % NF;
    if (fi > fj) continue;                 // upper fragments only; mirrored below
    // four independent accumulator chains over k (the DMMA latency, not its throughput, bounds a
    // single 8x8 fragment at this size), summed in a fixed order
    double c[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    const double* a = A + (fi * 8 + g) * P + t;
    const double* b = B + (fj * 8 + g) * P + t;
#pragma unroll
    for (int k = 0; k < DP; k += 16) {
#pragma unroll
      for (int u = 0; u < 4; ++u) dmma_8x8x4(c[u][0], c[u][1], a[k + 4 * u], b[k + 4 * u]);
    }
    const int r = fi * 8 + g, cc = fj * 8 + 2 * t;
    C[r * P + cc] = (c[0][0] + c[1][0]) + (c[2][0] + c[3][0]);
    C[r * P + cc + 1] = (c[0][1] + c[1][1]) + (c[2][1] + c[3][1]);
  }
  __syncthreads();
  // mirror: lower triangle (and the lower half of diagonal fragments) from the upper values
  for (int e = threadIdx.x; e < DP * DP; e += kSmallThreads) {
    const int i = e / DP, j = e % DP;
    if (i > j) C[i * P + j] = C[j * P + i];
  }
  __syncthreads();
}

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < kSmallThreads / 32; ++w) s += red[w];
  return s;
}

}  // namespace nsr
