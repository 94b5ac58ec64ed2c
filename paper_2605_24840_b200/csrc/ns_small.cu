// Small-d fast path (d <= 96): the whole Newton–Schulz loop of one problem in ONE CTA, with
// X, Y and Z = X Y resident in shared memory (SURVEY §8(a) a9 / K7 for configs[0]-sized problems).
// One launch per call (or per batch: one CTA per problem), no host round trips: the step count is
// decided inside the kernel by the same rule as ns_decide_kernel, so latency is the arithmetic
// (~2 x d^3 FMA per step on one SM's FP64 tensor pipe) instead of 3 launches + a status read per step.
//
// Products use DMMA m8n8k4 fragments read straight from row-major shared memory with a padded pitch
// (d_pad + 4 doubles: the 8 rows of a fragment land 32 B apart, conflict-free per half-warp).  Only the
// upper 8x8 fragments are computed; each is written with its mirror straight from registers, and the
// residual / update / trace are applied in the same epilogue, so one NS step is two products and two
// barriers (the earlier version ran separate mirror, residual and update passes over shared memory:
// 92 us for configs[0], most of it in those passes).
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "ns_internal.h"
#include "ns_ptx.cuh"
#include "ns_small.cuh"

#ifndef NS_SMALL_TRACE
#define NS_SMALL_TRACE 0   // 1: thread 0 records %globaltimer at phase boundaries (tools/small_trace.py)
#endif

namespace nsr {

#if NS_SMALL_TRACE
__device__ unsigned long long g_small_trace[256];   // [0] start, [1] init done, [2 + p] after product p (clock64);
                                                    // [128 + w], [160 + w]: warp w's DMMA loop end in
                                                    // products 0, 1; [250]: product counter
#define NS_STRACE(i) do { if (threadIdx.x == 0 && blockIdx.x == 0) g_small_trace[(i)] = clock64(); } while (0)
#else
#define NS_STRACE(i) do { } while (0)
#endif

// one warp per work unit (a pair of upper fragments sharing their A rows, see small_ns_product):
// 6 / 20 / 42 units for d_pad 32 / 64 / 96 (d_pad 96: 14 warps x 3 units, within the register file)
template <int DP>
__host__ __device__ constexpr int small_units() {
  int n = 0;
  for (int fi = 0; fi < DP / 8; ++fi) n += (DP / 8 - fi + 1) / 2;
  return n;
}
// Work-unit table (fi, fj) per warp slot w: single-fragment units (the last of each odd-length fragment
// row) first, then the pairs, so consecutive warps -- which sit on different SM sub-partitions with
// separate DMMA pipes -- share the singles.  Filled once per CTA (small_fill_units), read per product.
template <int DP>
__device__ __forceinline__ void small_fill_units(int2* tab) {
  constexpr int NF = DP / 8;
  constexpr int NS = NF / 2;               // single-fragment units: rows with an odd count NF - fi
  if (threadIdx.x != 0) return;
  int s = 0, pr = 0;
  for (int fi = 0; fi < NF; ++fi) {
    const int nu = (NF - fi + 1) / 2;
    for (int m = 0; m < nu; ++m) {
      const bool single = ((NF - fi) & 1) && m == nu - 1;
      tab[single ? s++ : NS + pr++] = make_int2(fi, fi + 2 * m);
    }
  }
}

// Row pitch (doubles) of the shared-memory matrices.  DP + 8 makes two fragment rows 16 banks apart, so
// a quarter-warp's 16-byte loads (rows g, g+1; k = 2t, 2t+1) are conflict-free; d_pad 96 keeps DP + 4
// (three 96 x 104 matrices would exceed the 227 KB shared-memory limit) and 8-byte loads.
template <int DP>
__host__ __device__ constexpr int small_pitch() { return DP == 96 ? DP + 4 : DP + 8; }

// CL = 1: one CTA per problem; CL = 2 (opt-in, NS_SMALL_CL=2): a cluster of two CTAs per problem,
// each taking every other work unit and storing its results into both CTAs' shared memory (DSMEM).
#ifndef NS_SMALL_QUAD
#define NS_SMALL_QUAD 1   // d_pad 64, one CTA: 2x2-fragment work units (see small_ns_product)
#endif
template <int DP, int CL = 1>
__host__ __device__ constexpr bool small_quad() { return NS_SMALL_QUAD && DP == 64 && CL == 1; }
template <int DP, int CL = 1>
__host__ __device__ constexpr int small_threads() {
  return small_quad<DP, CL>() ? 32 * 10
         : CL == 2 ? 32 * ((small_units<DP>() + 1) / 2)
                   : 32 * (small_units<DP>() <= 24 ? small_units<DP>() : (small_units<DP>() + 2) / 3);
}

__device__ __forceinline__ void st_cluster(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}

// Upper 8x8 fragments (fi <= fj) of C = A B^T for row-major smem operands with pitch DP+4, with the
// Newton–Schulz epilogue applied in registers (no separate mirror / residual / update passes):
//   MODE 0: C = A A^T = Y_j; writes the fragment and its mirror; returns this thread's share of
//           ||Y_j - I||_F^2 (diagonal fragments: elements c >= r only, off-diagonal weight 2).
//   MODE 1: C = ca X + cb (X Y) = X_{j+1} (X = A); writes it and its mirror; returns this thread's
//           share of tr X_{j+1}.
// Diagonal fragments store only c >= r and mirror those, so every stored matrix is bitwise symmetric.
// CL = 2: every store also goes to the peer CTA's copy (shared::cluster address = local + rdelta).
// Epilogue of one 8x8 fragment held as c[h] = C[r][c0 + h] (see small_ns_product).
template <int DP, int MODE, int CL>
__device__ __forceinline__ void small_frag_epilogue(const double (&c)[2], int r, int c0, bool diag,
                                                    const double* __restrict__ A, double* __restrict__ C, int d,
                                                    double ca, double cb, double& acc, uint32_t rdelta) {
  constexpr int P = small_pitch<DP>();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int cc = c0 + h;
    if (diag && cc < r) continue;          // lower half of a diagonal fragment: comes from the mirror
    double v = c[h];
    if (MODE == 0) {
      const double e = (cc == r && r < d) ? v - 1.0 : v;
      acc += (cc == r ? 1.0 : 2.0) * e * e;
    } else {
      v = fma(cb, v, ca * A[r * P + cc]);
      if (cc == r && r < d) acc += v;
    }
    C[r * P + cc] = v;
    if (cc != r) C[cc * P + r] = v;
    if constexpr (CL == 2) {
      st_cluster(smem_u32(C + r * P + cc) + rdelta, v);
      if (cc != r) st_cluster(smem_u32(C + cc * P + r) + rdelta, v);
    }
  }
}

// Upper part of C = A B^T for row-major smem operands with pitch DP+4, with the Newton–Schulz epilogue
// applied in registers (no separate mirror / residual / update passes):
//   MODE 0: C = A A^T = Y_j; writes each value and its mirror; returns this thread's share of
//           ||Y_j - I||_F^2 (diagonal fragments: elements c >= r only, off-diagonal weight 2).
//   MODE 1: C = ca X + cb (X Y) = X_{j+1} (X = A); writes it and its mirror; returns this thread's
//           share of tr X_{j+1}.
// Work unit = two horizontally adjacent upper fragments (fi, fj), (fi, fj+1) (the second absent at the
// end of a row), so each loaded A fragment feeds two DMMAs; one unit per warp (d_pad 96: two), which
// spreads the 8x8x4 DMMAs evenly over the four SM sub-partitions — one CTA is bound by the SM's FP64
// tensor path (64 FMA/clk).  Diagonal fragments store only c >= r and mirror those, so every stored
// matrix is bitwise symmetric.  CL = 2: CTA `rank` of the pair takes units rank, rank + 2, ...
template <int DP, int MODE, int CL>
__device__ __forceinline__ double small_ns_product(const double* __restrict__ A, const double* __restrict__ B,
                                                   double* __restrict__ C, int d, double ca, double cb,
                                                   const int2* __restrict__ units, int rank, uint32_t rdelta) {
  constexpr int P = small_pitch<DP>();
  constexpr bool VEC = ((2 * P) % 32) == 16;
  constexpr int NU = small_units<DP>();
  constexpr int NW = small_threads<DP, CL>() / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  double acc = 0.0;
  if constexpr (small_quad<DP, CL>()) {
    // d_pad 64: work unit = a 16x16 block of the upper triangle (2x2 fragments; on the diagonal the three
    // fragments with fi <= fj), one per warp: 4 shared-memory loads feed 8 DMMAs (pairs: 3 loads, 4 DMMAs) --
    // the pair units kept the shared-memory pipe ~85% busy inside a product and the DMMA pipe at ~74%.
    // Warps w = 0, 1, 4, 5 (SM sub-partitions 0, 1) take the 4 diagonal blocks (48 DMMAs per k sweep), the
    // other 6 warps the off-diagonal blocks (64): per sub-partition 160, 160, 128, 128 DMMAs.
    // (si, sj) of warp w: nibble w of these constants -- si 0 1 0 0 2 3 0 1 1 2, sj 0 1 1 2 2 3 3 2 3 3
    const int si = (int)((0x2110320010ull >> (4 * warp)) & 15), sj = (int)((0x3323322110ull >> (4 * warp)) & 15);
    const bool dg = si == sj;
    double c[4][2][2];                     // c[2 ia + ib][k-chain][h]
#pragma unroll
    for (int q = 0; q < 4; ++q) c[q][0][0] = c[q][0][1] = c[q][1][0] = c[q][1][1] = 0.0;
    const double* a0 = A + (16 * si + g) * P + 2 * t;
    const double* a1 = a0 + 8 * P;
    const double* b0 = B + (16 * sj + g) * P + 2 * t;
    const double* b1 = b0 + 8 * P;
#pragma unroll
    for (int k = 0; k < DP; k += 8) {
      const double2 x0 = *reinterpret_cast<const double2*>(a0 + k);
      const double2 x1 = *reinterpret_cast<const double2*>(a1 + k);
      const double2 y0 = *reinterpret_cast<const double2*>(b0 + k);
      const double2 y1 = *reinterpret_cast<const double2*>(b1 + k);
      // consecutive DMMAs share an operand register (A, B, A, ...): the operand reuse path, as in the tiled kernels
      dmma_8x8x4(c[0][0][0], c[0][0][1], x0.x, y0.x);
      dmma_8x8x4(c[1][0][0], c[1][0][1], x0.x, y1.x);
      dmma_8x8x4(c[3][0][0], c[3][0][1], x1.x, y1.x);
      if (!dg) dmma_8x8x4(c[2][0][0], c[2][0][1], x1.x, y0.x);
      dmma_8x8x4(c[0][1][0], c[0][1][1], x0.y, y0.y);
      dmma_8x8x4(c[1][1][0], c[1][1][1], x0.y, y1.y);
      dmma_8x8x4(c[3][1][0], c[3][1][1], x1.y, y1.y);
      if (!dg) dmma_8x8x4(c[2][1][0], c[2][1][1], x1.y, y0.y);
    }
#if NS_SMALL_TRACE
    if (lane == 0 && blockIdx.x == 0 && g_small_trace[250] < 2) g_small_trace[128 + 32 * (int)g_small_trace[250] + warp] = clock64();
#endif
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int ia = q >> 1, ib = q & 1;
      if (dg && ia > ib) continue;
      const double v[2] = {c[q][0][0] + c[q][1][0], c[q][0][1] + c[q][1][1]};
      small_frag_epilogue<DP, MODE, CL>(v, 16 * si + 8 * ia + g, 16 * sj + 8 * ib + 2 * t, dg && ia == ib, A, C, d,
                                        ca, cb, acc, rdelta);
    }
    return acc;
  }
  for (int w = CL * warp + rank; w < NU; w += CL * NW) {
    const int2 un = units[w];
    const int fi = un.x, fj = un.y;
    const bool two = (fj + 1 < DP / 8);
    double c[2][4][2];                     // c[fragment][k-chain][h]
#pragma unroll
    for (int f = 0; f < 2; ++f)
#pragma unroll
      for (int q = 0; q < 4; ++q) c[f][q][0] = c[f][q][1] = 0.0;
    if constexpr (VEC) {
      // k-permuted fragments: thread t supplies k = 2t (chain 0) and 2t+1 (chain 1) of each 8-wide k
      // block with one 16-byte load; both operands use the same permutation, so every product
      // A[i][k] B[j][k] still meets its partner (the summation order differs, not the sum's terms).
      // Odd 8-wide k blocks feed chains 2 and 3 (four independent accumulator chains per fragment).
      const double* a = A + (fi * 8 + g) * P + 2 * t;
      const double* b0 = B + (fj * 8 + g) * P + 2 * t;
      const double* b1 = b0 + 8 * P;
#pragma unroll
      for (int k = 0; k < DP; k += 16) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const double2 x = *reinterpret_cast<const double2*>(a + k + 8 * u);
          const double2 y0 = *reinterpret_cast<const double2*>(b0 + k + 8 * u);
          dmma_8x8x4(c[0][2 * u][0], c[0][2 * u][1], x.x, y0.x);
          dmma_8x8x4(c[0][2 * u + 1][0], c[0][2 * u + 1][1], x.y, y0.y);
          if (two) {
            const double2 y1 = *reinterpret_cast<const double2*>(b1 + k + 8 * u);
            dmma_8x8x4(c[1][2 * u][0], c[1][2 * u][1], x.x, y1.x);
            dmma_8x8x4(c[1][2 * u + 1][0], c[1][2 * u + 1][1], x.y, y1.y);
          }
        }
      }
    } else {
      const double* a = A + (fi * 8 + g) * P + t;
      const double* b0 = B + (fj * 8 + g) * P + t;
      const double* b1 = b0 + 8 * P;
#pragma unroll 4
      for (int k = 0; k < DP; k += 8) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const double x = a[k + 4 * q], y0 = b0[k + 4 * q];
          dmma_8x8x4(c[0][q][0], c[0][q][1], x, y0);
          if (two) dmma_8x8x4(c[1][q][0], c[1][q][1], x, b1[k + 4 * q]);
        }
      }
    }
#if NS_SMALL_TRACE
    if (lane == 0 && blockIdx.x == 0 && g_small_trace[250] < 2) g_small_trace[128 + 32 * (int)g_small_trace[250] + warp] = clock64();
#endif
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      if (f == 1 && !two) continue;
      const double v[2] = {(c[f][0][0] + c[f][1][0]) + (c[f][2][0] + c[f][3][0]),
                           (c[f][0][1] + c[f][1][1]) + (c[f][2][1] + c[f][3][1])};
      small_frag_epilogue<DP, MODE, CL>(v, fi * 8 + g, (fj + f) * 8 + 2 * t, fi == fj + f, A, C, d, ca, cb, acc,
                                        rdelta);
    }
  }
  return acc;
}

// CL = 1: one CTA per problem.  CL = 2: a cluster of two CTAs per problem: both hold X, Y, X_{j+1} in full,
// each computes half of every product's work units and stores the results into both copies over DSMEM; the
// per-warp partial sums go to both CTAs as well, so after each cluster barrier every warp of both CTAs forms
// the same fixed-order residual / trace and takes the same stop decision.  (configs[0]: the product's DMMA and
// shared-memory work per SM halves; the price is ~18 KB of DSMEM stores and one cluster barrier per product.)
template <int DP, int CL>
__global__ void __launch_bounds__(small_threads<DP, CL>(), 1)
    ns_small_kernel(const double* __restrict__ H, long long ldh, long long h_stride, const JobParams* __restrict__ jobs,
                    JobParams job0, LoopParams lp, double* __restrict__ R, long long ldr, long long r_stride,
                    DevState* __restrict__ state) {
  constexpr int P = small_pitch<DP>();
  constexpr int NT = small_threads<DP, CL>();
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) double sm[];
  double* X = sm;                  // X_j
  double* Xn = sm + DP * P;        // X_{j+1}
  double* Y = sm + 2 * DP * P;     // Y_j = X_j^2
  // warp partials [parity of j][rank][warp]: ||Y_j - I||_F^2 and tr X_j (double-buffered by step parity so a
  // fast warp of either CTA can never overwrite a slot another warp has yet to read)
  __shared__ double red_sq[2][CL][NW], red_tr[2][CL][NW];
  __shared__ int2 units[small_units<DP>()];
  NS_STRACE(0);
  small_fill_units<DP>(units);             // visible after the first barrier below
  const int rank = CL == 2 ? (int)cluster_ctarank() : 0;
  const int job = blockIdx.x / CL;
  const uint32_t rdelta = CL == 2 ? map_peer(smem_u32(sm), rank ^ 1) - smem_u32(sm) : 0u;
  const double* Hj = H + (long long)job * h_stride;
  const JobParams jp = jobs ? jobs[job] : job0;   // batch of one: parameters by value (no H2D copy)
  const double s = jp.s, alpha = jp.alpha;
  const int d = lp.d;
  const int wid = threadIdx.x >> 5, ln = threadIdx.x & 31;
  // X_0 = (H - sI)/alpha from the upper triangle, zero padded; tr X_0 partials.  Two passes, no integer
  // division: (1) warp w reads rows w, w + NW, ... of H's upper triangle (coalesced, every load of the
  // thread issued before the first use) into a pitch-(DP+1) staging copy in Y's buffer (free until the
  // first square); (2) element (i, j) takes staging[min][max] -- the transposed reads for j < i run down a
  // column of an odd-pitch array, conflict-free -- and is divided and stored row-wise into X.  (A flat-index
  // loop with per-element divisions and strided global reads of the lower half spent ~6400 cycles here.)
  // CL = 2: both CTAs form all of X_0; rank 1's trace share is zero.
  double tpart = 0.0;
  {
    constexpr int RPW = (DP + NW - 1) / NW, CPL = DP / 32, SP = DP + 1;
    double* Sg = Y;                        // staging, DP x SP <= DP x P
    double v[RPW][CPL];
#pragma unroll
    for (int q = 0; q < RPW; ++q)
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int i = wid + q * NW, jj = ln + 32 * c;
        v[q][c] = (i < d && jj < d && jj >= i) ? Hj[(long long)i * ldh + jj] : 0.0;
      }
#pragma unroll
    for (int q = 0; q < RPW; ++q)
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int i = wid + q * NW, jj = ln + 32 * c;
        if (i < DP) Sg[i * SP + jj] = v[q][c];
      }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < RPW; ++q)
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int i = wid + q * NW, jj = ln + 32 * c;
        if (i >= DP) continue;
        double x = 0.0;
        if (i < d && jj < d) {
          const double h = (jj >= i) ? Sg[i * SP + jj] : Sg[jj * SP + i];
          x = (i == jj) ? (h - s) / alpha : h / alpha;
          if (i == jj && rank == 0) tpart += x;
        }
        X[i * P + jj] = x;
      }
  }
  // tr X_0 partials into slot [0] (both CTAs' copies), then every CTA of the pair is past its init (the
  // staging in Y is dead) before any remote store lands
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tpart += __shfl_xor_sync(0xffffffffu, tpart, o);
  if (ln == 0) {
    red_tr[0][rank][wid] = tpart;
    if constexpr (CL == 2) st_cluster(smem_u32(&red_tr[0][rank][wid]) + rdelta, tpart);
  }
  if constexpr (CL == 2) cluster_sync_all();
  else __syncthreads();
  NS_STRACE(1);
  const double sqd = sqrt((double)d);
  // Stop rule of ns_decide_kernel, taken by EVERY warp from the same fixed-order sum (so all threads agree
  // without a second barrier and no update is computed past the decision): rho_j < tol is tested on the squared
  // residual a = r_j^2 against tol^2 (x d in the per-sqrt(d) mode) -- square roots and divisions are long FP64
  // sequences -- and re-tested exactly, as sqrt(a) (/ sqrt(d)) < tol, inside a +-1e-14 relative band around
  // the threshold, so the decision is bit-for-bit the one the rounded comparison takes.  Thread 0 alone forms
  // r_j = sqrt(a) for the SCALING_SUSPECT test and the result record, off the other warps' critical path.
  const double thr = lp.tol_mode ? lp.tol * lp.tol * (double)d : lp.tol * lp.tol;
  int j = 0, flags = 0;
  double r = 0.0, r_prev = 0.0, tr = 0.0;
  while (true) {
    const int par = j & 1;
    double part = small_ns_product<DP, 0, CL>(X, X, Y, d, 0.0, 0.0, units, rank, rdelta);   // Y_j, ||Y_j - I||^2 share
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (ln == 0) {
      red_sq[par][rank][wid] = part;
      if constexpr (CL == 2) st_cluster(smem_u32(&red_sq[par][rank][wid]) + rdelta, part);
    }
    if constexpr (CL == 2) cluster_sync_all();                     // Y_j complete in both CTAs, partials in
    else __syncthreads();                                          // Y_j complete, partials in red_sq
    NS_STRACE(2 + 2 * j);
#if NS_SMALL_TRACE
    if (threadIdx.x == 0 && blockIdx.x == 0 && g_small_trace[250] == 0) g_small_trace[250] = 1;   // stamps: products 0, 1
#endif
    double a = 0.0, b = 0.0;
    for (int e = ln; e < CL * NW; e += 32) {
      a += red_sq[par][e / NW][e % NW];
      b += red_tr[par][e / NW][e % NW];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    bool stop = false;
    if (!isfinite(a)) {
      stop = true;
    } else {
      bool conv = a < thr * (1.0 - 1e-14);
      if (!conv && a <= thr * (1.0 + 1e-14) && a > 0.0) {
        const double rr = sqrt(a);
        conv = (lp.tol_mode ? rr / sqd : rr) < lp.tol;
      }
      stop = conv || j >= lp.max_steps;
      if (threadIdx.x == 0) {
        const double rr = sqrt(a);
        if (j > 0 && rr > r_prev * (1.0 + 1e-12) + 1e-10 * sqd) flags |= 8;
        flags |= conv ? 1 : (j >= lp.max_steps ? 2 : 0);
        if (!stop) r_prev = rr;
      }
    }
    if (stop) {
      if (threadIdx.x == 0) {
        r = sqrt(a);
        if (!isfinite(r)) flags |= 16;
      }
      tr = b;
      break;
    }
    double tn = small_ns_product<DP, 1, CL>(X, Y, Xn, d, lp.ca, lp.cb, units, rank, rdelta);   // X_{j+1}
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tn += __shfl_xor_sync(0xffffffffu, tn, o);
    if (ln == 0) {
      red_tr[par ^ 1][rank][wid] = tn;
      if constexpr (CL == 2) st_cluster(smem_u32(&red_tr[par ^ 1][rank][wid]) + rdelta, tn);
    }
    if constexpr (CL == 2) cluster_sync_all();                     // X_{j+1} complete in both CTAs
    else __syncthreads();
    NS_STRACE(3 + 2 * j);
#if NS_SMALL_TRACE
    if (threadIdx.x == 0 && blockIdx.x == 0 && g_small_trace[250] == 1) g_small_trace[250] = 2;
#endif
    double* tmp = X;
    X = Xn;
    Xn = tmp;
    ++j;
  }
  // R = X_j (warp w: rows w, w + NW, ...; coalesced row stores, no integer division); CL = 2: rank r the rows
  // of parity r.  No remote access follows the last cluster barrier, so the two CTAs may exit independently.
  double* Rj = R + (long long)job * r_stride;
  for (int i = CL * wid + rank; i < d; i += CL * NW)
#pragma unroll
    for (int c = 0; c < DP / 32; ++c) {
      const int jj = ln + 32 * c;
      if (jj < d) Rj[(long long)i * ldr + jj] = X[i * P + jj];
    }
  NS_STRACE(100);
  if (threadIdx.x == 0 && rank == 0) {
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

// Diagnostics (NS_SMALL_TRACE builds): copy the phase stamps of the last traced launch to the host and clear them.
int small_trace_read(unsigned long long* out, int n) {
#if NS_SMALL_TRACE
  if (cudaMemcpyFromSymbol(out, g_small_trace, sizeof(unsigned long long) * (n < 256 ? n : 256)) != cudaSuccess) return -1;
  static const unsigned long long zero[256] = {};
  cudaMemcpyToSymbol(g_small_trace, zero, sizeof(zero));
  return n < 256 ? n : 256;
#else
  (void)out;
  (void)n;
  return 0;
#endif
}

int small_dpad(int d) { return d <= 32 ? 32 : d <= 64 ? 64 : d <= 96 ? 96 : 0; }

cudaError_t launch_small(const double* H, long long ldh, long long h_stride, const JobParams* jobs, JobParams job0,
                         LoopParams lp, double* R, long long ldr, long long r_stride, DevState* state, int batch,
                         cudaStream_t st) {
  static unsigned long long attr[6] = {0, 0, 0, 0, 0, 0};
  const int dp = small_dpad(lp.d);
  const size_t smem = (size_t)3 * dp * (dp == 96 ? dp + 4 : dp + 8) * sizeof(double);
  // NS_SMALL_CL=2: a single problem of d_pad 64 / 96 on a cluster of two CTAs (DSMEM exchange).  Measured equal to
  // one CTA at configs[0] (the halved DMMA phase, ~2000 instead of ~3100 cycles per product, is spent again on
  // ~18 KB of DSMEM stores and a cluster barrier per product), so one CTA per problem is the default.
  static const bool cl_env = [] {
    const char* e = getenv("NS_SMALL_CL");
    return e && e[0] == '2';
  }();
  const bool cl2 = cl_env && batch == 1 && dp >= 64;
  auto go = [&](auto kern, int threads, unsigned long long& a, int cl) -> cudaError_t {
    smem_attr(kern, (int)smem, a);
    if (cl == 1) {
      kern<<<batch, threads, smem, st>>>(H, ldh, h_stride, jobs, job0, lp, R, ldr, r_stride, state);
      return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(2 * batch);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, H, ldh, h_stride, jobs, job0, lp, R, ldr, r_stride, state);
  };
  switch (dp) {
    case 32:
      return go(ns_small_kernel<32, 1>, small_threads<32, 1>(), attr[0], 1);
    case 64:
      return cl2 ? go(ns_small_kernel<64, 2>, small_threads<64, 2>(), attr[1], 2)
                 : go(ns_small_kernel<64, 1>, small_threads<64, 1>(), attr[2], 1);
    case 96:
      return cl2 ? go(ns_small_kernel<96, 2>, small_threads<96, 2>(), attr[3], 2)
                 : go(ns_small_kernel<96, 1>, small_threads<96, 1>(), attr[4], 1);
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace nsr
