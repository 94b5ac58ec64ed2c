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

#include "ns_internal.h"
#include "ns_ptx.cuh"
#include "ns_small.cuh"

#ifndef NS_SMALL_SQ_MODE1
#define NS_SMALL_SQ_MODE1 0   // experiment: the square through the update's epilogue code (timing only)
#endif
#ifndef NS_SMALL_SQ_COPY
#define NS_SMALL_SQ_COPY 0   // experiment (tools/small_trace.py): the square reads its B operand from a copy of X
#endif
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

template <int DP>
__host__ __device__ constexpr int small_threads() { return 32 * (small_units<DP>() <= 24 ? small_units<DP>() : (small_units<DP>() + 2) / 3); }

// Upper 8x8 fragments (fi <= fj) of C = A B^T for row-major smem operands with pitch DP+4, with the
// Newton–Schulz epilogue applied in registers (no separate mirror / residual / update passes):
//   MODE 0: C = A A^T = Y_j; writes the fragment and its mirror; returns this thread's share of
//           ||Y_j - I||_F^2 (diagonal fragments: elements c >= r only, off-diagonal weight 2).
//   MODE 1: C = ca X + cb (X Y) = X_{j+1} (X = A); writes it and its mirror; returns this thread's
//           share of tr X_{j+1}.
// Diagonal fragments store only c >= r and mirror those, so every stored matrix is bitwise symmetric.
// Epilogue of one 8x8 fragment held as c[h] = C[r][c0 + h] (see small_ns_product).
template <int DP, int MODE>
__device__ __forceinline__ void small_frag_epilogue(const double (&c)[2], int r, int c0, bool diag,
                                                    const double* __restrict__ A, double* __restrict__ C, int d,
                                                    double ca, double cb, double& acc) {
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
// matrix is bitwise symmetric.
template <int DP, int MODE>
__device__ __forceinline__ double small_ns_product(const double* __restrict__ A, const double* __restrict__ B,
                                                   double* __restrict__ C, int d, double ca, double cb,
                                                   const int2* __restrict__ units) {
  constexpr int P = small_pitch<DP>();
  constexpr bool VEC = ((2 * P) % 32) == 16;
  constexpr int NU = small_units<DP>();
  constexpr int NW = small_threads<DP>() / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  double acc = 0.0;
  for (int w = warp; w < NU; w += NW) {
    const int2 un = units[w];
    const int fi = un.x, fj = un.y;
    const bool two = (fj + 1 < DP / 8);
    double c[2][2][2];                     // c[fragment][k-chain][h]
#pragma unroll
    for (int f = 0; f < 2; ++f)
#pragma unroll
      for (int q = 0; q < 2; ++q) c[f][q][0] = c[f][q][1] = 0.0;
    if constexpr (VEC) {
      // k-permuted fragments: thread t supplies k = 2t (chain 0) and 2t+1 (chain 1) of each 8-wide k
      // block with one 16-byte load; both operands use the same permutation, so every product
      // A[i][k] B[j][k] still meets its partner (the summation order differs, not the sum's terms).
      const double* a = A + (fi * 8 + g) * P + 2 * t;
      const double* b0 = B + (fj * 8 + g) * P + 2 * t;
      const double* b1 = b0 + 8 * P;
#pragma unroll 4
      for (int k = 0; k < DP; k += 8) {
        const double2 x = *reinterpret_cast<const double2*>(a + k);
        const double2 y0 = *reinterpret_cast<const double2*>(b0 + k);
        dmma_8x8x4(c[0][0][0], c[0][0][1], x.x, y0.x);
        dmma_8x8x4(c[0][1][0], c[0][1][1], x.y, y0.y);
        if (two) {
          const double2 y1 = *reinterpret_cast<const double2*>(b1 + k);
          dmma_8x8x4(c[1][0][0], c[1][0][1], x.x, y1.x);
          dmma_8x8x4(c[1][1][0], c[1][1][1], x.y, y1.y);
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
      const double v[2] = {c[f][0][0] + c[f][1][0], c[f][0][1] + c[f][1][1]};
      small_frag_epilogue<DP, MODE>(v, fi * 8 + g, (fj + f) * 8 + 2 * t, fi == fj + f, A, C, d, ca, cb, acc);
    }
  }
  return acc;
}

template <int DP>
__global__ void __launch_bounds__(small_threads<DP>(), 1)
    ns_small_kernel(const double* __restrict__ H, long long ldh, long long h_stride, const JobParams* __restrict__ jobs,
                    JobParams job0, LoopParams lp, double* __restrict__ R, long long ldr, long long r_stride,
                    DevState* __restrict__ state) {
  constexpr int P = small_pitch<DP>();
  constexpr int NT = small_threads<DP>();
  extern __shared__ __align__(16) double sm[];
  double* X = sm;                  // X_j
  double* Xn = sm + DP * P;        // X_{j+1}
  double* Y = sm + 2 * DP * P;     // Y_j = X_j^2
  __shared__ double red[NT / 32][2];
  __shared__ double dec_r, dec_tr;            // warp 0's stop decision of the current step
  __shared__ int dec_flags, dec_stop;
  __shared__ int2 units[small_units<DP>()];
  NS_STRACE(0);
  small_fill_units<DP>(units);             // visible after the first barrier below
  const int job = blockIdx.x;
  const double* Hj = H + (long long)job * h_stride;
  const JobParams jp = jobs ? jobs[job] : job0;   // batch of one: parameters by value (no H2D copy)
  const double s = jp.s, alpha = jp.alpha;
  const int d = lp.d;
  // X_0 = (H - sI)/alpha from the upper triangle, zero padded; tr X_0 partials.  Two passes, no integer
  // division: (1) warp w reads rows w, w + NW, ... of H's upper triangle (coalesced, every load of the
  // thread issued before the first use) into a pitch-(DP+1) staging copy in Y's buffer (free until the
  // first square); (2) element (i, j) takes staging[min][max] -- the transposed reads for j < i run down a
  // column of an odd-pitch array, conflict-free -- and is divided and stored row-wise into X.  (A flat-index
  // loop with per-element divisions and strided global reads of the lower half spent ~6400 cycles here.)
  double tpart = 0.0;
  {
    constexpr int NW = NT / 32, RPW = (DP + NW - 1) / NW, CPL = DP / 32, SP = DP + 1;
    double* Sg = Y;                        // staging, DP x SP <= DP x P
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    double v[RPW][CPL];
#pragma unroll
    for (int q = 0; q < RPW; ++q)
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int i = w + q * NW, jj = ln + 32 * c;
        v[q][c] = (i < d && jj < d && jj >= i) ? Hj[(long long)i * ldh + jj] : 0.0;
      }
#pragma unroll
    for (int q = 0; q < RPW; ++q)
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int i = w + q * NW, jj = ln + 32 * c;
        if (i < DP) Sg[i * SP + jj] = v[q][c];
      }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < RPW; ++q)
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int i = w + q * NW, jj = ln + 32 * c;
        if (i >= DP) continue;
        double x = 0.0;
        if (i < d && jj < d) {
          const double h = (jj >= i) ? Sg[i * SP + jj] : Sg[jj * SP + i];
          x = (i == jj) ? (h - s) / alpha : h / alpha;
          if (i == jj) tpart += x;
        }
        X[i * P + jj] = x;
      }
  }
  __syncthreads();
  NS_STRACE(1);
  const double sqd = sqrt((double)d);
  int j = 0, flags = 0;
  double r = 0.0, r_prev = 0.0, tr = 0.0;
  while (true) {
#if NS_SMALL_SQ_COPY
    // experiment: the square's B operand from a copy of X in Xn's (free) buffer instead of X itself
    for (int e = threadIdx.x; e < DP * P; e += NT) Xn[e] = X[e];
    __syncthreads();
    NS_STRACE(200 + j);
    double part = small_ns_product<DP, 0>(X, Xn, Y, d, 0.0, 0.0, units);
#elif NS_SMALL_SQ_MODE1
    // experiment: the square through the update's code path (epilogue ca = 0, cb = 1; no residual)
    double part = small_ns_product<DP, 1>(X, X, Y, d, 0.0, 1.0, units);
    part = 1.0;
#else
    double part = small_ns_product<DP, 0>(X, X, Y, d, 0.0, 0.0, units);   // Y_j = X_j^2, ||Y_j - I||_F^2 share
#endif
    // Stop rule (ns_decide_kernel's) evaluated once, by warp 0, instead of redundantly by every thread: the
    // square root, the division and the comparisons in all 20 warps cost ~1000 cycles of FP64 issue per step
    // (tools/small_trace.py).  Warp partials -> barrier (Y_j complete) -> warp 0 reduces in a fixed order and
    // decides -> barrier -> everyone reads the decision.
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      part += __shfl_xor_sync(0xffffffffu, part, o);
      tpart += __shfl_xor_sync(0xffffffffu, tpart, o);
    }
    if ((threadIdx.x & 31) == 0) {
      red[threadIdx.x >> 5][0] = part;
      red[threadIdx.x >> 5][1] = tpart;
    }
    __syncthreads();                                                // Y_j complete, partials in red
    NS_STRACE(2 + 2 * j);
#if NS_SMALL_TRACE
    if (threadIdx.x == 0 && blockIdx.x == 0 && g_small_trace[250] == 0) g_small_trace[250] = 1;   // stamps: products 0, 1
#endif
    if (threadIdx.x < 32) {
      double a = threadIdx.x < NT / 32 ? red[threadIdx.x][0] : 0.0;
      double b = threadIdx.x < NT / 32 ? red[threadIdx.x][1] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
      }
      if (threadIdx.x == 0) {
        const double rr = sqrt(a);
        int fl = flags, stop = 0;
        if (!isfinite(rr)) {
          fl |= 16;
          stop = 1;
        } else {
          if (j > 0 && rr > r_prev * (1.0 + 1e-12) + 1e-10 * sqd) fl |= 8;
          const double rho = lp.tol_mode ? rr / sqd : rr;
          if (rho < lp.tol) {
            fl |= 1;
            stop = 1;
          } else if (j >= lp.max_steps) {
            fl |= 2;
            stop = 1;
          }
        }
        dec_r = rr;
        dec_tr = b;
        dec_flags = fl;
        dec_stop = stop;
      }
    }
    // The update runs speculatively while warp 0 takes the decision (its sequential square root, division and
    // comparisons, ~1500 cycles, hide behind the other warps' DMMAs; warp 0 holds a single-fragment unit).
    // If the decision was to stop, X_j is returned and the extra X_{j+1} in Xn is simply not used.
    const double tpart_n = small_ns_product<DP, 1>(X, Y, Xn, d, lp.ca, lp.cb, units);   // ca X_j + cb X_j Y_j
    __syncthreads();                                                 // X_{j+1} complete, decision visible
    NS_STRACE(3 + 2 * j);
#if NS_SMALL_TRACE
    if (threadIdx.x == 0 && blockIdx.x == 0 && g_small_trace[250] == 1) g_small_trace[250] = 2;
#endif
    r = dec_r;
    tr = dec_tr;
    flags = dec_flags;
    if (dec_stop) break;
    tpart = tpart_n;
    double* tmp = X;
    X = Xn;
    Xn = tmp;
    r_prev = r;
    ++j;
  }
  // R = X_j (warp w: rows w, w + NW, ...; coalesced row stores, no integer division)
  double* Rj = R + (long long)job * r_stride;
  {
    constexpr int NW = NT / 32;
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    for (int i = w; i < d; i += NW)
#pragma unroll
      for (int c = 0; c < DP / 32; ++c) {
        const int jj = ln + 32 * c;
        if (jj < d) Rj[(long long)i * ldr + jj] = X[i * P + jj];
      }
  }
  NS_STRACE(100);
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
  static unsigned long long attr[3] = {0, 0, 0};
  const int dp = small_dpad(lp.d);
  const size_t smem = (size_t)3 * dp * (dp == 96 ? dp + 4 : dp + 8) * sizeof(double);
  switch (dp) {
    case 32:
      ns_small_kernel<32><<<batch, small_threads<32>(), smem, st>>>(H, ldh, h_stride, jobs, job0, lp, R, ldr, r_stride, state);
      break;
    case 64:
      smem_attr(ns_small_kernel<64>, (int)smem, attr[1]);
      ns_small_kernel<64><<<batch, small_threads<64>(), smem, st>>>(H, ldh, h_stride, jobs, job0, lp, R, ldr, r_stride, state);
      break;
    case 96:
      smem_attr(ns_small_kernel<96>, (int)smem, attr[2]);
      ns_small_kernel<96><<<batch, small_threads<96>(), smem, st>>>(H, ldh, h_stride, jobs, job0, lp, R, ldr, r_stride, state);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace nsr
