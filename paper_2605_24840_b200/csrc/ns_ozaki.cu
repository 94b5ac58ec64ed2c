// FP64-accurate products on the INT8 tensor cores (tcgen05 kind::i8) by the Ozaki splitting
// (SURVEY §8(f) N4 -- an arithmetic variant, not in the paper).
//
// Every operand row i is scaled by its own power of two and cut exactly into 7 signed 8-bit slices:
// N_ij = rint(x_ij 2^{54-e_i}) (e_i = frexp exponent of the row max, so |N| < 2^54) is written in
// balanced base 256, N = sum_{s=0..6} D^s 256^{6-s}, D^s in [-128, 127] (|D^0| <= 64).  Then
//     (P Q^T)_ij ~= 2^{e_i + f_j - 12} sum_{g=0}^{6} 2^{-8g} sum_{s+t=g} (D_P^s D_Q^t^T)_ij
// keeping the 28 slice pairs with s + t <= 6 (the dropped ones lie below ~2^-50 of |row| |col| per term;
// balanced digits keep the tails of small entries small -- floor-based unsigned tails do not).  Each
// slice product is EXACT in INT32; the seven group sums live in seven INT32 TMEM accumulators and are
// folded into FP64 registers every 16384 of K (7 x 16384 x 128^2 < 2^31, so any d), with exact
// conversions and power-of-two weights; one rounding per fold.
//
// CTA tile 128 x 64, 7 accumulators x 64 columns = 448 TMEM columns.  Stage = one 64-wide k-block of
// the 7 digits of both operands (7 x 8 KB + 7 x 4 KB, 64-B swizzle), 2 stages; warp 0 TMA, warp 1 MMA,
// warps 2..9 epilogue.  The B digit slabs lie back to back, so the pairs (sa, sb0..sb0+n-1) are ONE
// UMMA (M=128, N=64n <= 256, K=32) writing n adjacent group accumulators: 10 UMMAs per K=32 half
// instead of 28 (ncu: with 28 N=64 UMMAs the issuing warp, not the tensor pipe, was the limit).
// Symmetric outputs: tiles (I, J2) with J2*64 + 63 >= I*128; every element with j >= i is produced
// by exactly one tile, which writes it and its mirror (bitwise-symmetric output).
// Persistent launch (one CTA per SM walking the tile list): the producer prefetches the next tile and
// the MMA warp starts it while the epilogue writes the previous one from registers.
#include <algorithm>
#include <cmath>
#include <cstdint>

#include "ns_internal.h"
#include "ns_ptx.cuh"

namespace nsr {

// per-row exponent e_i (row max < 2^{e_i}) and S int8 slices; one block per row, grid.y = job
__global__ void __launch_bounds__(256) ns_ozaki_slice_kernel(const double* __restrict__ X, int8_t* __restrict__ slices,
                                                             int* __restrict__ expo, int d_pad) {
  __shared__ double red[8];
  const int row = blockIdx.x, job = blockIdx.y;
  const long long nn = (long long)d_pad * d_pad;
  const double* x = X + (long long)job * nn + (long long)row * d_pad;
  double m = 0.0;
  for (int j = threadIdx.x; j < d_pad; j += 256) {
    const double a = fabs(x[j]);
    m = (a > m || a != a) ? a : m;               // NaN / Inf propagate (fmax would drop a NaN)
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double b = __shfl_xor_sync(0xffffffffu, m, o);
    m = (b > m || b != b) ? b : m;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  double mm = 0.0;
  for (int w = 0; w < 8; ++w) mm = (red[w] > mm || red[w] != red[w]) ? red[w] : mm;
  int e = 0;
  if (!isfinite(mm)) e = kOzBadRow;                  // non-finite row: the products of this row come out NaN
  else if (mm > 0.0) frexp(mm, &e);                 // mm = f 2^e, f in [0.5, 1)  =>  |x_ij| < 2^e
  if (threadIdx.x == 0) expo[(long long)job * d_pad + row] = e;
  if (e == kOzBadRow) {
    int8_t* o0 = slices + (long long)job * kOzSlices * nn + (long long)row * d_pad;
    for (int j = threadIdx.x; j < d_pad; j += 256)
      for (int q = 0; q < kOzSlices; ++q) o0[(long long)q * nn + j] = 0;
    return;
  }
  int8_t* out = slices + (long long)job * kOzSlices * nn + (long long)row * d_pad;
  for (int j = threadIdx.x; j < d_pad; j += 256) {
    // N = x 2^{54-e} rounded to an integer (|N| < 2^54), written in balanced base 256:
    // N = sum_s D_s 256^{6-s}, D_1..D_6 in [-128, 127], |D_0| <= 64.  A small |x| has zero leading
    // digits, so every slice-pair product stays relative to the operands' own magnitudes.
    long long N = (long long)rint(ldexp(x[j], 54 - e));
#pragma unroll
    for (int q = kOzSlices - 1; q >= 1; --q) {
      const long long D = ((N + 128) & 255) - 128;
      out[(long long)q * nn + j] = (int8_t)D;
      N = (N - D) >> 8;                          // exact
    }
    out[j] = (int8_t)N;
  }
}

// The same exponent and digits with one warp per row (8 rows per block): for small d_pad (the batched
// configs) a 256-thread block per 256-element row was mostly block scheduling and barrier overhead.
__global__ void __launch_bounds__(256) ns_ozaki_slice_rows_kernel(const double* __restrict__ X,
                                                                  int8_t* __restrict__ slices, int* __restrict__ expo,
                                                                  int d_pad) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), job = blockIdx.y, lane = threadIdx.x & 31;
  const long long nn = (long long)d_pad * d_pad;
  const double* x = X + (long long)job * nn + (long long)row * d_pad;
  double m = 0.0;
  for (int j = lane; j < d_pad; j += 32) {
    const double a = fabs(x[j]);
    m = (a > m || a != a) ? a : m;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double b = __shfl_xor_sync(0xffffffffu, m, o);
    m = (b > m || b != b) ? b : m;
  }
  int e = 0;
  if (!isfinite(m)) e = kOzBadRow;
  else if (m > 0.0) frexp(m, &e);
  if (lane == 0) expo[(long long)job * d_pad + row] = e;
  int8_t* out = slices + (long long)job * kOzSlices * nn + (long long)row * d_pad;
  if (e == kOzBadRow) {
    for (int j = lane; j < d_pad; j += 32)
      for (int q = 0; q < kOzSlices; ++q) out[(long long)q * nn + j] = 0;
    return;
  }
  for (int j = lane; j < d_pad; j += 32) {
    long long N = (long long)rint(ldexp(x[j], 54 - e));
#pragma unroll
    for (int q = kOzSlices - 1; q >= 1; --q) {
      const long long D = ((N + 128) & 255) - 128;
      out[(long long)q * nn + j] = (int8_t)D;
      N = (N - D) >> 8;
    }
    out[j] = (int8_t)N;
  }
}

// TMA load delivered to the same shared-memory offset in every CTA of `mask` (cluster multicast); each
// destination CTA's barrier at `bar`'s offset receives the bytes.
__device__ __forceinline__ void tma_load_3d_mc(void* dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
// arrive (once) on the barrier at this offset in every CTA of `mask` when this thread's prior tcgen05
// operations complete
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// K-major operand, kOzKH-byte swizzle: rows of kOzKH bytes, 8-row atoms 8 * kOzKH bytes apart (SBO),
// version 1; layout type 4 = 64-byte swizzle, 6 = 32-byte swizzle.
__device__ __forceinline__ uint64_t sdesc_k64(uint32_t saddr) {
  constexpr uint64_t sbo = (8ull * kOzKH) >> 4, lay = kOzKH == 32 ? 6ull : 4ull;
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | (1ull << 16) | (sbo << 32) | (1ull << 46) | (lay << 61);
}

template <int MODE, bool MC, int G>
__global__ void __launch_bounds__(kOzThreads, 1)
    ns_ozaki_product_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                            const OzParams p, int n_items) {
  // Persistent: CTA b processes work items b, b + gridDim.x, ... (item = job * n_tiles + tile).  The
  // stage ring, the chunk handshake and their phase bits run on across tiles, so the producer streams
  // the next tile's k-blocks while the epilogue drains this one, and the MMA warp starts the next tile
  // as soon as the accumulators are in registers (the epilogue writes C straight from registers:
  // there is no staging buffer to wait for).
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kOzStages * kOzStageBytes);
  uint64_t* empty = full + kOzStages;
  uint64_t* tfull = empty + kOzStages;     // chunk accumulated (MMA -> epilogue)
  uint64_t* tempty = tfull + 1;            // chunk folded into FP64 registers (epilogue -> MMA)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  double* stage_base = reinterpret_cast<double*>(smem + kOzStages * kOzStageBytes + 256);   // 4 x [32][17]
  __shared__ double red[8];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_chunks = (p.nkb + kOzChunkKb - 1) / kOzChunkKb;
  // MC (cluster of 2): work items are 128 x 128 tiles walked per cluster; CTA `rank` takes the 64-column
  // half 2 J + rank.  The 7 A digit slabs of a k-block are shared: each CTA loads about half of them with
  // TMA multicast into both CTAs' shared memory (half the A traffic from L2 per CTA).
  const int rank = MC ? (int)cluster_ctarank() : 0;
  const int item0 = MC ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int istride = MC ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  auto tile_of = [&](int item, int job) -> int2 {
    const int2 t = p.tiles[item - job * p.n_tiles];
    return MC ? make_int2(t.x, 2 * t.y + rank) : t;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kOzStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC ? 2 : 1);   // MC: both CTAs' MMA warps release a slot (their A halves are shared)
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 8);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  if (MC) cluster_sync_all();              // peer barriers initialised before any multicast / remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      uint32_t kbg = 0;                    // stages issued by this CTA so far (ring position)
      constexpr int kSub = 64 / kOzKH;     // stages per 64-wide k-block
      for (int item = item0; item < n_items; item += istride) {
        const int job = item / p.n_tiles;
        if (p.state != nullptr && p.state[job].done) continue;
        const int2 tile = tile_of(item, job);
        for (int kb = 0; kb < p.nkb * kSub; ++kb, ++kbg) {
          const int kx = p.kb0 * 64 + kb * kOzKH;   // k coordinate (bytes) of this stage
          const int s = kbg % kOzStages;
          if (kbg >= kOzStages) mbar_wait(&empty[s], ((kbg / kOzStages) & 1u) ^ 1u);
          uint8_t* st = smem + s * kOzStageBytes;
          mbar_arrive_expect_tx(&full[s], kOzStageBytes);
          if (MC) {
#pragma unroll
            for (int q = 0; q < kOzSlices; ++q)
              if ((q & 1) == rank)
                tma_load_3d_mc(st + q * kOzSlabA, &tmA, kx, tile.x * kTile, job * kOzSlices + q,
                               &full[s], 0x3);
          } else {
#pragma unroll
            for (int q = 0; q < kOzSlices; ++q)
              tma_load_3d(st + q * kOzSlabA, &tmA, kx, tile.x * kTile, job * kOzSlices + q, &full[s]);
          }
#pragma unroll
          for (int q = 0; q < kOzSlices; ++q)
            tma_load_3d(st + kOzSlices * kOzSlabA + q * kOzSlabB, &tmB, kx, tile.y * 64, job * kOzSlices + q,
                        &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // idesc: D=S32 (bits 4-5 = 2), A/B signed int8 (bits 7-9 / 10-12 = 1), K-major, M=128 (N set per MMA).
    const uint32_t idesc_base = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kTile >> 4) << 24);
    uint32_t kbg = 0, cg = 0;              // k-blocks / chunks consumed by this CTA so far
    for (int item = item0; item < n_items; item += istride) {
      const int job = item / p.n_tiles;
      if (p.state != nullptr && p.state[job].done) continue;
      for (int c = 0; c < n_chunks; ++c, ++cg) {
        if (cg >= 1) mbar_wait(tempty, (cg - 1) & 1u);   // accumulators folded by the epilogue
        tc_fence_after();
        constexpr int kSub = 64 / kOzKH;
        const int kb0 = c * kOzChunkKb * kSub, kb1 = min(p.nkb * kSub, kb0 + kOzChunkKb * kSub);
        for (int kb = kb0; kb < kb1; ++kb, ++kbg) {
          const int s = kbg % kOzStages;
          mbar_wait(&full[s], (kbg / kOzStages) & 1u);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t a0 = smem_u32(smem + s * kOzStageBytes);
            if (!p.dbg) {
            const uint32_t b0 = a0 + kOzSlices * kOzSlabA;
            const uint32_t first = (kb == kb0) ? 0u : 1u;
            // Digit pairs (sa, sb), sb = sb0 .. sb0+n-1, share the A digit: the B digit slabs are stored
            // back to back (64 rows each), so rows [64 sb0, 64 (sb0+n)) form ONE K-major operand of
            // N = 64 n whose output columns are exactly the group accumulators sa+sb0 .. sa+sb0+n-1.
            // 28 pairs (34 with the eighth group) become 10 (15) UMMAs (N = 64..256) per K=32 half.
#pragma unroll
            for (int h = 0; h < kOzKH / 32; ++h) {
#pragma unroll
              for (int sa = 0; sa < kOzSlices; ++sa) {
                const int nb = min(kOzSlices, G - sa);   // B digits paired with A digit sa (s + t < G)
                auto issue = [&](int sb, int n, uint32_t acc) {
                  const uint32_t idesc = idesc_base | ((uint32_t)(64 * n >> 3) << 17);
                  umma_i8(tmem + (uint32_t)(64 * (sa + sb)), sdesc_k64(a0 + sa * kOzSlabA + 32 * h),
                          sdesc_k64(b0 + sb * kOzSlabB + 32 * h), idesc, acc);
                };
#pragma unroll
                for (int sb0 = 0; sb0 < nb; sb0 += 4) {
                  const int n = min(4, nb - sb0);
                  const uint32_t acc = (sa == 0 && h == 0) ? first : 1u;
                  if (G > kOzSlices && sa == 1 && sb0 + n == nb) {
                    // the eighth group (s + t = 7) is first written by pair (1, 6): that column block
                    // starts the chunk on its own UMMA, the rest of the range accumulates
                    if (n > 1) issue(sb0, n - 1, acc);
                    issue(nb - 1, 1, h == 0 ? first : 1u);
                  } else {
                    issue(sb0, n, acc);
                  }
                }
              }
            }
            }
            if (MC) umma_commit_mc(&empty[s], 0x3);   // release the slot in both CTAs
            else umma_commit(&empty[s]);
            if (kb == kb1 - 1) umma_commit(tfull);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ---------------- epilogue warps 2..9: TMEM lane quadrant q = warp % 4, column half hc ----------------
    const int q = warp & 3, hc = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    const int ew = warp - 2;               // 0..7
    uint32_t cg = 0;
    for (int item = item0; item < n_items; item += istride) {
      const int job = item / p.n_tiles;
      if (p.state != nullptr && p.state[job].done) continue;
      const int2 tile = tile_of(item, job);
      double acc[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) acc[c] = 0.0;
      for (int ch = 0; ch < n_chunks; ++ch, ++cg) {
        mbar_wait(tfull, cg & 1u);
        tc_fence_after();
#pragma unroll 1
        for (int g = G - 1; g >= 0; --g) {      // smallest weights first
          const double w = ldexp(1.0, -8 * g);
          uint32_t v[32];
          tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(g * 64 + hc * 32), v);   // one wait per group
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[i] = fma((double)(int)v[i], w, acc[i]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty);   // TMEM free: the MMA warp may start the next chunk / tile
      }
      // ---- write-out from registers (row r of the tile, columns 32 hc .. 32 hc + 31) ----
      const long long base = (long long)job * p.job_stride;
      const long long ld = p.ld;
      double* C = p.C + base;
      const int i0 = tile.x * kTile, j0 = tile.y * 64 + hc * 32, gi = i0 + r;
      const int er = p.expP[(long long)job * ld + gi];
      const int* ecol = p.expQ + (long long)job * ld + j0;
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        // times 2^(er + ec - 12): one multiply by the power of two built from its bits (ldexp only when
        // that power is outside the normal range, i.e. for extreme operand scales)
        const int ex = er + ecol[c] - 12;
        acc[c] = (ex >= -1022 && ex <= 1023) ? acc[c] * __hiloint2double((ex + 1023) << 20, 0)
                 : (er == kOzBadRow || ecol[c] == kOzBadRow) ? __longlong_as_double(0x7ff8000000000000LL)   // NaN
                                                             : ldexp(acc[c], ex);
      }
      double part = 0.0;
      const double* X = p.Xold + base;
      double* stg = stage_base + ew * (32 * 17);   // this warp's 32 x 16 staging block (pitch 17)
      // 16-column blocks: values (MODE 1: from X_j, read 16 at a time ahead of any store) are computed
      // per thread (= row), mirrors go straight out (lanes = consecutive rows of the mirror: coalesced),
      // and the row-major part is transposed through the staging block so every store instruction
      // writes two full 128-byte row segments.
      // K segments (d > 16384): segments before the last store raw partial sums of the owned elements in
      // C; the last adds them back and runs the mode epilogue (launches are stream-ordered)
      const bool fin = (p.pm == 0 || p.pm == 3);
      if (p.pm >= 2) {
#pragma unroll
        for (int cb = 0; cb < 2; ++cb) {
          double pbuf[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int gj = j0 + 16 * cb + u;
            pbuf[u] = (MODE == 2 || gj >= gi) ? C[(long long)gi * ld + gj] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 16; ++u) acc[16 * cb + u] += pbuf[u];
        }
      }
#pragma unroll
      for (int cb = 0; cb < 2; ++cb) {
        double xbuf[16];
        if (MODE == 1 && fin) {
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int gj = j0 + 16 * cb + u;
            xbuf[u] = (gj >= gi) ? X[(long long)gi * ld + gj] : 0.0;
          }
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int c = 16 * cb + u, gj = j0 + c;
          double v = acc[c];
          if (MODE != 2 && gj >= gi && fin) {   // element owned by this tile (written with its mirror)
            if (MODE == 1) {
              v = fma(p.cb, v, p.ca * xbuf[u]);
              if (gi == gj && gi < p.d) {
                v += p.cc;
                part += v;
              }
            } else {
              if (gj > gi) part += 2.0 * v * v;
              else {
                const double e = (gi < p.d) ? v - 1.0 : v;
                part += e * e;
              }
            }
            if (gj > gi) C[(long long)gj * ld + gi] = v;
          }
          stg[lane * 17 + u] = v;
        }
        __syncwarp();
#pragma unroll 4
        for (int rr = 0; rr < 32; rr += 2) {
          const int row = rr + (lane >> 4), col = lane & 15;
          const int gi2 = i0 + q * 32 + row, gj2 = j0 + 16 * cb + col;
          if (MODE == 2 || gj2 >= gi2) C[(long long)gi2 * ld + gj2] = stg[row * 17 + col];
        }
        __syncwarp();
      }
      if (MODE != 2 && fin) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) red[ew] = part;
        named_bar_sync(1, 256);
        if (ew == 0 && lane == 0) {
          double sum = 0.0;
#pragma unroll
          for (int w = 0; w < 8; ++w) sum += red[w];
          const int i0t = tile.x * kTile, j0t = tile.y * 64;
          if (MODE == 0)
            p.partial[(long long)job * (MC ? 2 * p.n_tiles : p.n_tiles) + (item - job * p.n_tiles) * (MC ? 2 : 1) + rank] = sum;
          else if (j0t <= i0t + kTile - 1 && j0t + 63 >= i0t) p.partial[(long long)job * (2 * (p.ld / kTile)) + tile.y] = sum;
        }
        named_bar_sync(1, 256);              // red[] is reused by the next tile
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (MC) cluster_sync_all();              // no multicast into, or arrive on, a CTA that has left
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// Cluster-of-2 Ozaki products (A digits multicast) on by default; NS_OZ_MC=0 selects single CTAs.
bool use_oz_mc() {
  static const bool on = [] {
    const char* e = getenv("NS_OZ_MC");
    return !(e && e[0] == '0');
  }();
  return on;
}

cudaError_t launch_ozaki_slice(const double* X, int8_t* slices, int* expo, int d_pad, int batch, cudaStream_t st) {
  if (d_pad <= 2048) {
    dim3 grid(d_pad / 8, batch);
    ns_ozaki_slice_rows_kernel<<<grid, 256, 0, st>>>(X, slices, expo, d_pad);
  } else {
    dim3 grid(d_pad, batch);
    ns_ozaki_slice_kernel<<<grid, 256, 0, st>>>(X, slices, expo, d_pad);
  }
  return cudaGetLastError();
}

// one persistent launch of the product kernel; MC: clusters of 2 CTAs on 128 x 128 tiles (p.tiles holds
// (I, J) of 128-column blocks)
template <int MODE, bool MC, int G>
static cudaError_t oz_launch(const CUtensorMap& tmA, const CUtensorMap& tmB, const OzParams& p, int n_items, dim3 grid,
                             cudaStream_t st) {
  static unsigned long long attr = 0;
  smem_attr(ns_ozaki_product_kernel<MODE, MC, G>, kOzSmemBytes, attr);
  if (MC) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kOzThreads);
    cfg.dynamicSmemBytes = kOzSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, ns_ozaki_product_kernel<MODE, MC, G>, tmA, tmB, p, n_items);
  }
  ns_ozaki_product_kernel<MODE, MC, G><<<grid, kOzThreads, kOzSmemBytes, st>>>(tmA, tmB, p, n_items);
  return cudaGetLastError();
}

cudaError_t launch_ozaki_product(const CUtensorMap& tmA, const CUtensorMap& tmB, const OzParams& p, int batch,
                                 cudaStream_t st) {
  static int n_sm = 0;
  if (n_sm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (n_sm <= 0) n_sm = 148;
  }
  static const int dbg = [] {
    const char* e = getenv("NS_OZ_DBG");
    return e ? atoi(e) : 0;
  }();
  if (dbg != p.dbg) {
    OzParams q = p;
    q.dbg = dbg;
    return launch_ozaki_product(tmA, tmB, q, batch, st);
  }
  if (p.pm == 0 && p.nkb > kOzSegKb) {
    // K segments of kOzSegKb k-blocks, one launch each: every segment streams a K range that the
    // concurrently working CTAs share in L2 (whole-K tiles at d = 49152 drifted apart: 40% L2 hits,
    // HBM-bound); partial sums go through C (stream-ordered launches)
    const int nseg = (p.nkb + kOzSegKb - 1) / kOzSegKb;
    for (int sgi = 0; sgi < nseg; ++sgi) {
      OzParams q = p;
      q.kb0 = sgi * kOzSegKb;
      q.nkb = std::min(kOzSegKb, p.nkb - q.kb0);
      q.pm = (sgi == 0) ? 1 : (sgi == nseg - 1 ? 3 : 2);
      const cudaError_t e = launch_ozaki_product(tmA, tmB, q, batch, st);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  const int n_items = p.n_tiles * batch;
  const bool mc = use_oz_mc();
  const dim3 grid = mc ? dim3(2 * std::min(n_items, n_sm / 2)) : dim3(std::min(n_items, n_sm));
  const int g8 = (p.groups > kOzSlices) ? 1 : 0;
  switch ((p.mode == 0 ? 0 : p.mode == 1 ? 1 : 2) * 4 + (mc ? 2 : 0) + g8) {
    case 0: return oz_launch<0, false, 7>(tmA, tmB, p, n_items, grid, st);
    case 1: return oz_launch<0, false, 8>(tmA, tmB, p, n_items, grid, st);
    case 2: return oz_launch<0, true, 7>(tmA, tmB, p, n_items, grid, st);
    case 3: return oz_launch<0, true, 8>(tmA, tmB, p, n_items, grid, st);
    case 4: return oz_launch<1, false, 7>(tmA, tmB, p, n_items, grid, st);
    case 5: return oz_launch<1, false, 8>(tmA, tmB, p, n_items, grid, st);
    case 6: return oz_launch<1, true, 7>(tmA, tmB, p, n_items, grid, st);
    case 7: return oz_launch<1, true, 8>(tmA, tmB, p, n_items, grid, st);
    case 8: return oz_launch<2, false, 7>(tmA, tmB, p, n_items, grid, st);
    case 9: return oz_launch<2, false, 8>(tmA, tmB, p, n_items, grid, st);
    case 10: return oz_launch<2, true, 7>(tmA, tmB, p, n_items, grid, st);
    default: return oz_launch<2, true, 8>(tmA, tmB, p, n_items, grid, st);
  }
}

}  // namespace nsr
