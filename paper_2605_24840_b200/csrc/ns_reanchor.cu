// Re-anchoring of the mixed-precision iterate (reading C16).
//
// After the BF16x3 phase the iterate X~ is close to a reflector, but its invariant subspace is
// rotated by O(split rounding): at a reflector S the Newton–Schulz map has derivative
// Df(S)[E] = (E - SES)/2, which is 0 on errors commuting with S and the identity on errors
// anticommuting with S, so FP64 polishing alone converges to sgn(X~) instead of sgn(A)
// (A = X_0 = (H - sI)/alpha).  The anticommuting error E is recovered from the FP64
// commutator with A:  C = [A, X~] = M - M^T with M = A X~,  and for X~ = S + E,
//     X~ C ~ |A| E + E |A|        (|A| = S A ~ sym(M)),
// so E solves the Lyapunov-type equation  |A| E + E |A| = F := sym(X~ C)  (SPD on symmetric
// matrices, eigenvalues |mu_i| + |mu_j| >= 2 gamma).  It is solved by conjugate gradients with
// the operator applied through the tcgen05 BF16x3 core (W = |A| P, L(P) = W + W^T), then
// X~ <- X~ - E and the FP64 Newton–Schulz steps continue.
//
// This file holds the HBM-bound elementwise/transposing kernels of that solve; the products
// (M = A X~, X~ C in FP64 DMMA; |A| P in BF16x3) reuse the contraction kernels.  Every
// reduction writes per-block partials that a single block sums in a fixed order, so the
// solve is bitwise deterministic.
#include <cuda_bf16.h>

#include <cstdint>

#include "ns_internal.h"
#include "ns_ptx.cuh"

namespace nsr {

__device__ __forceinline__ void split_bf16_r(double x, uint16_t& hi, uint16_t& lo) {
  const __nv_bfloat16 h = __double2bfloat16(x);
  const __nv_bfloat16 l = __double2bfloat16(x - (double)__bfloat162float(h));
  hi = __bfloat16_as_ushort(h);
  lo = __bfloat16_as_ushort(l);
}

__device__ __forceinline__ uint32_t tf32_bits_r(float f) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(f));
  return r;
}

// hi/lo planes of one element (bf16 or tf32-as-fp32 layout), plane stride n
template <bool TF32>
__device__ __forceinline__ void put_planes(double x, void* planes, long long i, long long n) {
  if (TF32) {
    const uint32_t h = tf32_bits_r((float)x);
    const uint32_t l = tf32_bits_r((float)(x - (double)__uint_as_float(h)));
    static_cast<uint32_t*>(planes)[i] = h;
    static_cast<uint32_t*>(planes)[n + i] = l;
  } else {
    uint16_t h, l;
    split_bf16_r(x, h, l);
    static_cast<uint16_t*>(planes)[i] = h;
    static_cast<uint16_t*>(planes)[n + i] = l;
  }
}

// fixed-order block reduction of one double per thread (blockDim = 256) -> out[blockIdx]
__device__ __forceinline__ void block_partial(double v, double* out) {
  __shared__ double red[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += red[w];
    out[blockIdx.x] = s;
  }
}

// Upper 32x32 tile pair (bi <= bj) for a linear block index over nb(nb+1)/2 pairs.
__device__ __forceinline__ void tile_pair(int b, int nb, int& bi, int& bj) {
  // row bi has nb - bi pairs; walk rows (nb <= 2048, cheap)
  int r = 0;
  while (b >= nb - r) {
    b -= nb - r;
    ++r;
  }
  bi = r;
  bj = r + b;
}

// C = M - M^T,  |A| = (M + M^T)/2 -> bf16 hi/lo planes (the CG operator's left factor).
template <bool TF32>
__global__ void __launch_bounds__(256) ns_commutator_kernel(const double* __restrict__ M, double* __restrict__ C,
                                                            void* __restrict__ abs_planes, int d_pad,
                                                            double* __restrict__ partial) {
  __shared__ double ta[32][33], tb[32][33];
  const int nb = d_pad / 32;
  int bi, bj;
  tile_pair(blockIdx.x, nb, bi, bj);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const long long np = (long long)d_pad * d_pad;
  for (int y = ty; y < 32; y += 8) {
    ta[y][tx] = M[(long long)(bi * 32 + y) * d_pad + bj * 32 + tx];
    tb[y][tx] = M[(long long)(bj * 32 + y) * d_pad + bi * 32 + tx];
  }
  __syncthreads();
  double acc = 0.0;
  for (int y = ty; y < 32; y += 8) {
    // element (bi*32+y, bj*32+tx): M_ij = ta[y][tx], M_ji = tb[tx][y]
    const double mij = ta[y][tx], mji = tb[tx][y];
    const long long g1 = (long long)(bi * 32 + y) * d_pad + bj * 32 + tx;
    const long long g2 = (long long)(bj * 32 + y) * d_pad + bi * 32 + tx;
    C[g1] = mij - mji;
    acc += (bi == bj ? 1.0 : 2.0) * (mij - mji) * (mij - mji);   // ||C||_F^2: the mirror tile counts once more
    put_planes<TF32>(0.5 * (mij + mji), abs_planes, g1, np);
    if (bi != bj) {
      const double nij = tb[y][tx], nji = ta[tx][y];   // element (bj*32+y, bi*32+tx)
      C[g2] = nij - nji;
      put_planes<TF32>(0.5 * (nij + nji), abs_planes, g2, np);
    }
  }
  if (partial != nullptr) block_partial(acc, partial);
}

// F = -(F' + F'^T)/2 with F' = X~ C^T = -X~ C;  R = P = F, E = 0;  partial <R, R>.
__global__ void __launch_bounds__(256) ns_cg_init_kernel(const double* __restrict__ Fp, double* __restrict__ R,
                                                         double* __restrict__ P, double* __restrict__ E,
                                                         double* __restrict__ partial, int d_pad) {
  __shared__ double ta[32][33], tb[32][33];
  const int nb = d_pad / 32;
  int bi, bj;
  tile_pair(blockIdx.x, nb, bi, bj);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int y = ty; y < 32; y += 8) {
    ta[y][tx] = Fp[(long long)(bi * 32 + y) * d_pad + bj * 32 + tx];
    tb[y][tx] = Fp[(long long)(bj * 32 + y) * d_pad + bi * 32 + tx];
  }
  __syncthreads();
  double acc = 0.0;
  for (int y = ty; y < 32; y += 8) {
    const double f1 = -0.5 * (ta[y][tx] + tb[tx][y]);
    const long long g1 = (long long)(bi * 32 + y) * d_pad + bj * 32 + tx;
    R[g1] = f1;
    P[g1] = f1;
    E[g1] = 0.0;
    acc += (bi == bj ? 1.0 : 2.0) * f1 * f1;   // <R,R> over the full matrix: mirror counted once more
    if (bi != bj) {
      const double f2 = -0.5 * (tb[y][tx] + ta[tx][y]);
      const long long g2 = (long long)(bj * 32 + y) * d_pad + bi * 32 + tx;
      R[g2] = f2;
      P[g2] = f2;
      E[g2] = 0.0;
    }
  }
  block_partial(acc, partial);
}

// partial <P, W> over all entries (grid-stride, fixed grid kEwBlocks).
__global__ void __launch_bounds__(256) ns_cg_pw_kernel(const double* __restrict__ P, const double* __restrict__ W,
                                                       double* __restrict__ partial, long long n,
                                                       const CgScalars* __restrict__ sc) {
  if (sc->done) return;
  double acc = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    acc = fma(P[i], W[i], acc);
  block_partial(acc, partial);
}

// which = 0: rr = rr0 = sum (tol2 set by the host);  1: pw = sum, alpha = rr / (2 pw);
// 2: beta = sum / rr, rr = sum, done once rr <= tol2 rr0 (the remaining launches of the solve return at once).
__global__ void __launch_bounds__(256) ns_cg_scalar_kernel(CgScalars* sc, const double* __restrict__ partial, int n,
                                                           int which, double tol2) {
  __shared__ double red[8];
  if (which != 0 && sc->done) return;
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) s += partial[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x != 0) return;
  double t = 0.0;
  for (int w = 0; w < 8; ++w) t += red[w];
  if (which == 0) {
    sc->rr = t;
    sc->rr0 = t;
    sc->tol2 = tol2;
    sc->done = (t == 0.0) ? 1 : 0;
    sc->iters = 0;
  } else if (which == 1) {
    sc->pw = t;
    sc->alpha = (t != 0.0) ? sc->rr / (2.0 * t) : 0.0;   // <P, L(P)> = <P, W + W^T> = 2 <P, W>
  } else {
    sc->beta = (sc->rr != 0.0) ? t / sc->rr : 0.0;
    sc->rr = t;
    sc->iters += 1;
    if (!(t > sc->tol2 * sc->rr0)) sc->done = 1;
  }
}

// E += alpha P;  R -= alpha (W + W^T);  partial <R, R>  (tile pairs for the transpose of W).
__global__ void __launch_bounds__(256) ns_cg_update_kernel(double* __restrict__ E, double* __restrict__ R,
                                                           const double* __restrict__ P, const double* __restrict__ W,
                                                           const CgScalars* __restrict__ sc,
                                                           double* __restrict__ partial, int d_pad) {
  __shared__ double ta[32][33], tb[32][33];
  if (sc->done) return;
  const int nb = d_pad / 32;
  int bi, bj;
  tile_pair(blockIdx.x, nb, bi, bj);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const double alpha = sc->alpha;
  for (int y = ty; y < 32; y += 8) {
    ta[y][tx] = W[(long long)(bi * 32 + y) * d_pad + bj * 32 + tx];
    tb[y][tx] = W[(long long)(bj * 32 + y) * d_pad + bi * 32 + tx];
  }
  __syncthreads();
  double acc = 0.0;
  for (int y = ty; y < 32; y += 8) {
    const long long g1 = (long long)(bi * 32 + y) * d_pad + bj * 32 + tx;
    E[g1] = fma(alpha, P[g1], E[g1]);
    const double r1 = fma(-alpha, ta[y][tx] + tb[tx][y], R[g1]);
    R[g1] = r1;
    acc += (bi == bj ? 1.0 : 2.0) * r1 * r1;
    if (bi != bj) {
      const long long g2 = (long long)(bj * 32 + y) * d_pad + bi * 32 + tx;
      E[g2] = fma(alpha, P[g2], E[g2]);
      R[g2] = fma(-alpha, tb[y][tx] + ta[tx][y], R[g2]);
    }
  }
  block_partial(acc, partial);
}

// P = R + beta P, and the bf16 hi/lo planes of the new P (right factor of W = |A| P).
template <bool TF32>
__global__ void __launch_bounds__(256) ns_cg_direction_kernel(double* __restrict__ P, const double* __restrict__ R,
                                                              const CgScalars* __restrict__ sc,
                                                              void* __restrict__ planes, long long n) {
  if (sc->done) return;
  const double beta = sc->beta;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double p = fma(beta, P[i], R[i]);
    P[i] = p;
    put_planes<TF32>(p, planes, i, n);
  }
}

__global__ void __launch_bounds__(256) ns_apply_correction_kernel(double* __restrict__ X, const double* __restrict__ E,
                                                                  long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    X[i] -= E[i];
}

// ------------------------------------------------------------------ launchers
static int n_pairs(int d_pad) {
  const int nb = d_pad / 32;
  return nb * (nb + 1) / 2;
}

cudaError_t launch_commutator(const double* M, double* C, void* abs_planes, int d_pad, cudaStream_t st, bool tf32,
                              double* partial, int* n_partial) {
  if (n_partial) *n_partial = n_pairs(d_pad);
  if (tf32) ns_commutator_kernel<true><<<n_pairs(d_pad), 256, 0, st>>>(M, C, abs_planes, d_pad, partial);
  else ns_commutator_kernel<false><<<n_pairs(d_pad), 256, 0, st>>>(M, C, abs_planes, d_pad, partial);
  return cudaGetLastError();
}

cudaError_t launch_cg_init(const double* Fp, double* R, double* P, double* E, double* partial, int d_pad,
                           cudaStream_t st, int* n_partial) {
  *n_partial = n_pairs(d_pad);
  ns_cg_init_kernel<<<n_pairs(d_pad), 256, 0, st>>>(Fp, R, P, E, partial, d_pad);
  return cudaGetLastError();
}

cudaError_t launch_cg_pw(const double* P, const double* W, double* partial, int d_pad, cudaStream_t st,
                         const CgScalars* sc) {
  ns_cg_pw_kernel<<<kEwBlocks, 256, 0, st>>>(P, W, partial, (long long)d_pad * d_pad, sc);
  return cudaGetLastError();
}

cudaError_t launch_cg_scalar(CgScalars* sc, const double* partial, int n_partial, int which, cudaStream_t st,
                             double tol2) {
  ns_cg_scalar_kernel<<<1, 256, 0, st>>>(sc, partial, n_partial, which, tol2);
  return cudaGetLastError();
}

cudaError_t launch_cg_update(double* E, double* R, const double* P, const double* W, const CgScalars* sc,
                             double* partial, int d_pad, cudaStream_t st, int* n_partial) {
  *n_partial = n_pairs(d_pad);
  ns_cg_update_kernel<<<n_pairs(d_pad), 256, 0, st>>>(E, R, P, W, sc, partial, d_pad);
  return cudaGetLastError();
}

cudaError_t launch_cg_direction(double* P, const double* R, const CgScalars* sc, void* p_planes, int d_pad,
                                cudaStream_t st, bool tf32) {
  if (tf32) ns_cg_direction_kernel<true><<<kEwBlocks, 256, 0, st>>>(P, R, sc, p_planes, (long long)d_pad * d_pad);
  else ns_cg_direction_kernel<false><<<kEwBlocks, 256, 0, st>>>(P, R, sc, p_planes, (long long)d_pad * d_pad);
  return cudaGetLastError();
}

cudaError_t launch_apply_correction(double* X, const double* E, int d_pad, cudaStream_t st) {
  ns_apply_correction_kernel<<<kEwBlocks, 256, 0, st>>>(X, E, (long long)d_pad * d_pad);
  return cudaGetLastError();
}

}  // namespace nsr
