// Mixed-precision (BF16x3 on tcgen05) contraction for the early Newton–Schulz steps
// (BASELINE north_star subsystem (1): "a mixed path (BF16x3 split with FP32 accumulate for
// the early contracting steps, then FP64 polishing steps)").
//
// Each FP64 operand X is kept in FP64 and mirrored into two BF16 planes, X = X_hi + X_lo + O(2^-17|X|).
// A product P Q^T is formed as P_hi Q_lo^T + P_lo Q_hi^T + P_hi Q_hi^T (the lo*lo term is below
// the FP32 accumulation floor), i.e. ONE tcgen05 GEMM over an extended K of 3*d, accumulated in
// FP32 in tensor memory.  The epilogue converts to FP64 and applies the same fused steps as the
// FP64 kernel (Y + residual, NS update + trace, bitwise-symmetric mirrored writes), and also
// re-emits the BF16 planes of its output for the next product.
//
// CTA = 10 warps: warp 0 TMA producer, warp 1 MMA issuer (one elected lane; owns the TMEM
// allocation), warps 2..9 epilogue (warp w reads TMEM lane quadrant w % 4, column half (w-2)/4).
// 128x128 output tile, UMMA M=128 N=128 K=16, 3-stage ring of 64 KB: each stage brings the hi and lo
// slabs of both operands for one 64-wide k-block (each byte fetched once; the kernel is L2-bandwidth
// bound) and feeds 12 UMMAs.  K is cut into chunks of kMxChunkKb*64; each chunk accumulates
// in FP32 into one of two 128-column TMEM buffers while the epilogue folds the previous chunk into
// FP64 registers, so FP32 accumulation error is bounded by the chunk length (C16 accuracy budget).
#include <cuda_bf16.h>

#include <cmath>
#include <cstdint>

#include "ns_internal.h"
#include "ns_ptx.cuh"

namespace nsr {

__device__ __forceinline__ void split_bf16(double x, uint16_t& hi, uint16_t& lo) {
  const __nv_bfloat16 h = __double2bfloat16(x);
  const double r = x - (double)__bfloat162float(h);
  const __nv_bfloat16 l = __double2bfloat16(r);
  hi = __bfloat16_as_ushort(h);
  lo = __bfloat16_as_ushort(l);
}

// TF32 split: hi = tf32(x) (10 explicit mantissa bits, stored as an fp32 bit pattern), lo = tf32(x - hi).
__device__ __forceinline__ uint32_t to_tf32_bits(float f) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(f));
  return r;
}
__device__ __forceinline__ void split_tf32(double x, uint32_t& hi, uint32_t& lo) {
  hi = to_tf32_bits((float)x);
  lo = to_tf32_bits((float)(x - (double)__uint_as_float(hi)));
}

template <bool TF32>
__device__ __forceinline__ void split_plane(double x, void* planes, long long i, long long n) {
  if (TF32) {
    uint32_t h, l;
    split_tf32(x, h, l);
    static_cast<uint32_t*>(planes)[i] = h;
    static_cast<uint32_t*>(planes)[n + i] = l;
  } else {
    uint16_t h, l;
    split_bf16(x, h, l);
    static_cast<uint16_t*>(planes)[i] = h;
    static_cast<uint16_t*>(planes)[n + i] = l;
  }
}

template <bool TF32>
__global__ void __launch_bounds__(256) ns_split_planes_kernel(const double* __restrict__ X, void* __restrict__ planes,
                                                              long long n_per_job, int batch) {
  const long long total = n_per_job * batch;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long job = i / n_per_job, e = i - job * n_per_job;
    void* base = TF32 ? (void*)(static_cast<uint32_t*>(planes) + job * 2 * n_per_job)
                      : (void*)(static_cast<uint16_t*>(planes) + job * 2 * n_per_job);
    split_plane<TF32>(X[i], base, e, n_per_job);
  }
}

__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Epilogue writes of one 128x128 output tile (I, J) staged in S[128][kEpiPitch] (FP64), by the 8
// epilogue warps (threads 64..319): C (+ its hi/lo planes), mirrors, residual / trace partials.
// `part_idx` is the tile's slot in the per-tile residual partials (MODE 0); `write` = false makes a
// tile contribute nothing (2-CTA pairs: a tile below the diagonal or beyond d_pad).
template <int MODE, bool TF32>
__device__ __forceinline__ void mx_tile_epilogue(double* S, int I, int J, int job, int part_idx, bool write,
                                                 const MxParams& p, double* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (!write) {
    if (MODE != 2 && lane == 0) red[warp - 2] = 0.0;
    named_bar_sync(1, kMxEpiThreads);
    if (MODE == 0 && threadIdx.x == 64) p.partial[(long long)job * p.n_tiles + part_idx] = 0.0;
    return;
  }
    const int tid = threadIdx.x - 64;       // 0..255
    const long long ld = p.ld;
    const long long base = (long long)job * p.job_stride;
    double* C = p.C + base;
    const long long nplane = (long long)p.ld * p.ld;
    void* Ph = nullptr;
    if (p.Cplanes) Ph = TF32 ? (void*)(static_cast<uint32_t*>(p.Cplanes) + (long long)job * 2 * nplane)
                             : (void*)(static_cast<uint16_t*>(p.Cplanes) + (long long)job * 2 * nplane);
    const bool diag = (I == J);
    double part = 0.0;
    auto put = [&](long long gidx, double v) {
      C[gidx] = v;
      if (Ph) split_plane<TF32>(v, Ph, gidx, nplane);
    };
    if (MODE == 2) {
      for (int idx = tid; idx < kTile * kTile; idx += kMxEpiThreads) {
        const int rr = idx >> 7, cc = idx & 127;
        put((long long)(I * kTile + rr) * ld + J * kTile + cc, S[rr * kEpiPitch + cc]);
      }
    } else if (MODE == 0) {
      if (!diag) {
        for (int idx = tid; idx < kTile * kTile; idx += kMxEpiThreads) {
          const int rr = idx >> 7, cc = idx & 127;
          const double v = S[rr * kEpiPitch + cc];
          put((long long)(I * kTile + rr) * ld + J * kTile + cc, v);
          part += v * v;
        }
        part *= 2.0;
        for (int idx = tid; idx < kTile * kTile; idx += kMxEpiThreads) {
          const int rr = idx >> 7, cc = idx & 127;
          put((long long)(J * kTile + rr) * ld + I * kTile + cc, S[cc * kEpiPitch + rr]);
        }
      } else {
        for (int idx = tid; idx < kTile * kTile; idx += kMxEpiThreads) {
          const int rr = idx >> 7, cc = idx & 127;
          const double v = (rr <= cc) ? S[rr * kEpiPitch + cc] : S[cc * kEpiPitch + rr];
          put((long long)(I * kTile + rr) * ld + I * kTile + cc, v);
          if (rr < cc) {
            part += 2.0 * v * v;
          } else if (rr == cc) {
            const double e = (I * kTile + rr < p.d) ? v - 1.0 : v;
            part += e * e;
          }
        }
      }
    } else {  // MODE 1: X_{j+1} = 1.5 X_j - 0.5 Z
      const double* X = p.Xold + base;
      if (!diag) {
        for (int idx = tid; idx < kTile * kTile; idx += kMxEpiThreads) {
          const int rr = idx >> 7, cc = idx & 127;
          const long long g = (long long)(I * kTile + rr) * ld + J * kTile + cc;
          const double v = fma(-0.5, S[rr * kEpiPitch + cc], 1.5 * X[g]);
          put(g, v);
          S[rr * kEpiPitch + cc] = v;
        }
        named_bar_sync(1, kMxEpiThreads);
        for (int idx = tid; idx < kTile * kTile; idx += kMxEpiThreads) {
          const int rr = idx >> 7, cc = idx & 127;
          put((long long)(J * kTile + rr) * ld + I * kTile + cc, S[cc * kEpiPitch + rr]);
        }
      } else {
        for (int idx = tid; idx < kTile * kTile; idx += kMxEpiThreads) {
          const int rr = idx >> 7, cc = idx & 127;
          if (rr <= cc) {
            const long long g = (long long)(I * kTile + rr) * ld + I * kTile + cc;
            const double v = fma(-0.5, S[rr * kEpiPitch + cc], 1.5 * X[g]);
            S[rr * kEpiPitch + cc] = v;
            if (rr == cc && I * kTile + rr < p.d) part += v;
          }
        }
        named_bar_sync(1, kMxEpiThreads);
        for (int idx = tid; idx < kTile * kTile; idx += kMxEpiThreads) {
          const int rr = idx >> 7, cc = idx & 127;
          put((long long)(I * kTile + rr) * ld + I * kTile + cc,
              (rr <= cc) ? S[rr * kEpiPitch + cc] : S[cc * kEpiPitch + rr]);
        }
      }
    }
    if (MODE != 2) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (lane == 0) red[warp - 2] = part;
      named_bar_sync(1, kMxEpiThreads);
      if (tid == 0) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < kMxEpiWarps; ++w) s += red[w];
        if (MODE == 0) p.partial[(long long)job * p.n_tiles + part_idx] = s;
        else if (diag) p.partial[(long long)job * (p.ld / kTile) + I] = s;
      }
    }
  }

template <int MODE, bool TF32>
__global__ void __launch_bounds__(kMxThreads, 1)
    ns_mx_product_kernel(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmQ,
                         const MxParams p) {
  constexpr int kKB = TF32 ? 32 : kMxBK;   // elements per 128-byte k-block row
  const int job = blockIdx.y;
  if (p.state != nullptr && (p.state[job].done || p.state[job].sw)) return;   // low-precision phase over
  if (p.skip != nullptr && *p.skip) return;                                    // CG solve already converged

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // stage s holds four 16 KB slabs: A_hi, A_lo, B_hi, B_lo (128 rows x 64 bf16 each, 128-B swizzle)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kMxStages * kMxStageBytes);
  uint64_t* empty = full + kMxStages;
  uint64_t* tfull = empty + kMxStages;     // [2] accumulator chunk ready (MMA -> epilogue)
  uint64_t* tempty = tfull + 2;            // [2] accumulator drained (epilogue -> MMA)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ double red[kMxEpiWarps];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int2 tile = p.tiles[blockIdx.x];
  const int I = tile.x, J = tile.y;
  const int nkb_total = p.nkb;
  constexpr int kChunk = TF32 ? kMxChunkKb / 2 : kMxChunkKb;   // same K per FP32 chunk in elements x bytes
  const int n_chunks = (nkb_total + kChunk - 1) / kChunk;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kMxEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 2 * kTile);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmP);
      tma_prefetch_desc(&tmQ);
      for (int kb = 0; kb < nkb_total; ++kb) {
        const int s = kb % kMxStages;
        const uint32_t use = kb / kMxStages;
        if (kb >= kMxStages) mbar_wait(&empty[s], (use & 1u) ^ 1u);
        uint8_t* st = smem + s * kMxStageBytes;
        mbar_arrive_expect_tx(&full[s], kMxStageBytes);
        tma_load_3d(st + 0 * kMxSlab, &tmP, kb * kKB, I * kTile, 2 * job + 0, &full[s]);   // P_hi
        tma_load_3d(st + 1 * kMxSlab, &tmP, kb * kKB, I * kTile, 2 * job + 1, &full[s]);   // P_lo
        tma_load_3d(st + 2 * kMxSlab, &tmQ, kb * kKB, J * kTile, 2 * job + 0, &full[s]);   // Q_hi
        tma_load_3d(st + 3 * kMxSlab, &tmQ, kb * kKB, J * kTile, 2 * job + 1, &full[s]);   // Q_lo
      }
    }
  } else if (warp == 1) {
    // idesc: D=F32 (bits 4-5 = 1), A=B=BF16 (1) or TF32 (2) (bits 7-9, 10-12), K-major, N=128, M=128
    constexpr uint32_t fmt = TF32 ? 2u : 1u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(kTile >> 3) << 17) |
                           ((uint32_t)(kTile >> 4) << 24);
    // K is cut into chunks of kMxChunkKb k-blocks; each chunk accumulates in FP32 into one of two TMEM
    // buffers, and the epilogue warps fold finished chunks into FP64 registers (FP32 accumulation error
    // then grows with the chunk length, not with 3*d).
    for (int c = 0; c < n_chunks; ++c) {
      const int b = c & 1;
      if (c >= 2) mbar_wait(&tempty[b], static_cast<uint32_t>((c >> 1) - 1) & 1u);
      tc_fence_after();
      const uint32_t acc = tmem + (uint32_t)(b * kTile);
      const int kb0 = c * kChunk, kb1 = min(nkb_total, kb0 + kChunk);
      for (int kb = kb0; kb < kb1; ++kb) {
        const int s = kb % kMxStages;
        mbar_wait(&full[s], static_cast<uint32_t>(kb / kMxStages) & 1u);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t ahi = smem_u32(smem + s * kMxStageBytes), alo = ahi + kMxSlab;
          const uint32_t bhi = ahi + 2 * kMxSlab, blo = ahi + 3 * kMxSlab;
          // the three split terms, small ones first: P_hi Q_lo^T + P_lo Q_hi^T + P_hi Q_hi^T
          // 4 UMMAs per 128-byte k-block row (K = 16 bf16 or 8 tf32 = 32 bytes each)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (TF32) umma_tf32(acc, sdesc_k128(ahi + k * 32), sdesc_k128(blo + k * 32), idesc, (kb != kb0) || (k != 0));
            else umma_bf16(acc, sdesc_k128(ahi + k * 32), sdesc_k128(blo + k * 32), idesc, (kb != kb0) || (k != 0));
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (TF32) umma_tf32(acc, sdesc_k128(alo + k * 32), sdesc_k128(bhi + k * 32), idesc, 1u);
            else umma_bf16(acc, sdesc_k128(alo + k * 32), sdesc_k128(bhi + k * 32), idesc, 1u);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (TF32) umma_tf32(acc, sdesc_k128(ahi + k * 32), sdesc_k128(bhi + k * 32), idesc, 1u);
            else umma_bf16(acc, sdesc_k128(ahi + k * 32), sdesc_k128(bhi + k * 32), idesc, 1u);
          }
          umma_commit(&empty[s]);
          if (kb == kb1 - 1) umma_commit(&tfull[b]);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------- epilogue: fold FP32 chunks into FP64 registers ----------------
    const int q = warp & 3;                        // TMEM lane quadrant of this warp
    const int h = (warp - 2) >> 2;                 // column half: 0 -> cols 0..63, 1 -> 64..127
    const int r = q * 32 + lane;                   // tile row owned by this thread
    double accd[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) accd[i] = 0.0;
    for (int c = 0; c < n_chunks; ++c) {
      const int b = c & 1;
      mbar_wait(&tfull[b], static_cast<uint32_t>(c >> 1) & 1u);
      tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * kTile + h * 64 + c0), v);
#pragma unroll
        for (int i = 0; i < 16; ++i) accd[c0 + i] += (double)__uint_as_float(v[i]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
    }
    // the ring is idle once the last chunk landed: stage the FP64 tile for the coalesced passes
    double* S = reinterpret_cast<double*>(smem);   // [128][kEpiPitch]
#pragma unroll
    for (int i = 0; i < 64; ++i) S[r * kEpiPitch + h * 64 + i] = accd[i];
  }
  // all roles: ring no longer in use (epilogue wrote S only after the last MMA completed)
  tc_fence_before();
  __syncthreads();

  if (warp >= 2)
    mx_tile_epilogue<MODE, TF32>(reinterpret_cast<double*>(smem), I, J, job, blockIdx.x, true, p, red);
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 2 * kTile);
}

__device__ __forceinline__ void umma_f16_cg2(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_tf32_cg2(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 2-SM split-precision product: the CTA pair of a 2-CTA cluster computes the 256 x 128 tile
// rows [256 I2, 256 I2 + 256) x cols [128 J, 128 J + 128) with M=256 UMMAs (cta_group::2) issued by the
// even CTA.  Each CTA stages its own 128 P rows and half (64 rows) of the 128 Q rows, so the shared-
// memory traffic per MAC is 3/4 of the one-SM kernel's (B read once for two 128-row halves) and a
// 4-stage ring fits.  Both CTAs' TMA loads complete on the leader's full barrier (which expects both
// CTAs' bytes); the leader's MMA commits multicast to both CTAs' empty / accumulator-full barriers; both
// CTAs' epilogue warps release a TMEM buffer on the leader's tempty barrier.  Each CTA then writes its
// own 128 x 128 tile (I = 2 I2 + rank, J) with the one-SM epilogue.
template <int MODE, bool TF32>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kMxThreads, 1)
    ns_mx2_product_kernel(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmQ,
                          const MxParams p) {
  constexpr int kKB = TF32 ? 32 : kMxBK;
  const int job = blockIdx.y;
  if (p.state != nullptr && (p.state[job].done || p.state[job].sw)) return;   // same for both CTAs
  if (p.skip != nullptr && *p.skip) return;                                    // CG solve already converged

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kMx2Stages * kMx2StageBytes);
  uint64_t* empty = full + kMx2Stages;
  uint64_t* tfull = empty + kMx2Stages;    // [2]
  uint64_t* tempty = tfull + 2;            // [2], used in the leader: 2 x 8 epilogue warps arrive
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ double red[kMxEpiWarps];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  unsigned long long t_start = 0;
  if (p.trace != nullptr && threadIdx.x == 64) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  const int2 pt = p.tiles[blockIdx.x >> 1];
  const int I = 2 * pt.x + (int)rank, J = pt.y;
  constexpr int kChunk = TF32 ? kMxChunkKb / 2 : kMxChunkKb;
  const int nkb_total = p.nkb;
  const int n_chunks = (nkb_total + kChunk - 1) / kChunk;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMx2Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * kMxEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_cg2(tmem_slot, 2 * kTile);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();                      // peer barriers initialised before any remote signal
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmP);
      tma_prefetch_desc(&tmQ);
      long long pw = 0;
      for (int kb = 0; kb < nkb_total; ++kb) {
        const int s = kb % kMx2Stages;
        if (kb >= kMx2Stages) {
          const long long w0 = p.trace ? clock64() : 0;
          mbar_wait(&empty[s], ((kb / kMx2Stages) & 1u) ^ 1u);
          if (p.trace) pw += clock64() - w0;
        }
        uint8_t* st = smem + s * kMx2StageBytes;
        if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * kMx2StageBytes);
        const uint32_t fb = map_peer(smem_u32(&full[s]), 0);
        tma_load_3d_cg2(st, &tmP, kb * kKB, I * kTile, 2 * job + 0, fb);                                // P_hi
        tma_load_3d_cg2(st + kMx2SlabA, &tmP, kb * kKB, I * kTile, 2 * job + 1, fb);                    // P_lo
        tma_load_3d_cg2(st + 2 * kMx2SlabA, &tmQ, kb * kKB, J * kTile + 64 * (int)rank, 2 * job + 0, fb);  // Q_hi half
        tma_load_3d_cg2(st + 2 * kMx2SlabA + kMx2SlabB, &tmQ, kb * kKB, J * kTile + 64 * (int)rank, 2 * job + 1, fb);
      }
      if (p.trace) p.trace[((long long)blockIdx.y * gridDim.x + blockIdx.x) * 12 + 6] = pw;
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // idesc: D=F32, A=B=BF16 (1) or TF32 (2), K-major, N=128, M=256 (cta_group::2)
      constexpr uint32_t fmt = TF32 ? 2u : 1u;
      const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(kTile >> 3) << 17) |
                             ((uint32_t)(256 >> 4) << 24);
      long long fw = 0, tw = 0;
      const long long m0 = p.trace ? clock64() : 0;
      for (int c = 0; c < n_chunks; ++c) {
        const int b = c & 1;
        if (c >= 2) {
          const long long w0 = p.trace ? clock64() : 0;
          mbar_wait(&tempty[b], static_cast<uint32_t>((c >> 1) - 1) & 1u);
          if (p.trace) tw += clock64() - w0;
        }
        tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)(b * kTile);
        const int kb0 = c * kChunk, kb1 = min(nkb_total, kb0 + kChunk);
        for (int kb = kb0; kb < kb1; ++kb) {
          const int s = kb % kMx2Stages;
          const long long w0 = p.trace ? clock64() : 0;
          mbar_wait(&full[s], static_cast<uint32_t>(kb / kMx2Stages) & 1u);
          if (p.trace) fw += clock64() - w0;
          tc_fence_after();
          if (elect_one()) {
            const uint32_t ahi = smem_u32(smem + s * kMx2StageBytes), alo = ahi + kMx2SlabA;
            const uint32_t bhi = ahi + 2 * kMx2SlabA, blo = bhi + kMx2SlabB;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if (TF32) umma_tf32_cg2(acc, sdesc_k128(ahi + k * 32), sdesc_k128(blo + k * 32), idesc, (kb != kb0) || (k != 0));
              else umma_f16_cg2(acc, sdesc_k128(ahi + k * 32), sdesc_k128(blo + k * 32), idesc, (kb != kb0) || (k != 0));
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if (TF32) umma_tf32_cg2(acc, sdesc_k128(alo + k * 32), sdesc_k128(bhi + k * 32), idesc, 1u);
              else umma_f16_cg2(acc, sdesc_k128(alo + k * 32), sdesc_k128(bhi + k * 32), idesc, 1u);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if (TF32) umma_tf32_cg2(acc, sdesc_k128(ahi + k * 32), sdesc_k128(bhi + k * 32), idesc, 1u);
              else umma_f16_cg2(acc, sdesc_k128(ahi + k * 32), sdesc_k128(bhi + k * 32), idesc, 1u);
            }
            umma_commit_cg2_mc(&empty[s], 3);
            if (kb == kb1 - 1) umma_commit_cg2_mc(&tfull[b], 3);
          }
          __syncwarp();
        }
      }
      if (p.trace && lane == 0) {
        const long long sl = ((long long)blockIdx.y * gridDim.x + blockIdx.x) * 12;
        p.trace[sl + 4] = fw;
        p.trace[sl + 5] = clock64() - m0;
        p.trace[sl + 7] = tw;
      }
    }
  } else {
    const int q = warp & 3, h = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    const uint32_t te0 = map_peer(smem_u32(&tempty[0]), 0), te1 = map_peer(smem_u32(&tempty[1]), 0);
    double accd[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) accd[i] = 0.0;
    long long ew = 0, ef = 0;
    for (int c = 0; c < n_chunks; ++c) {
      const int b = c & 1;
      const long long w0 = p.trace ? clock64() : 0;
      mbar_wait(&tfull[b], static_cast<uint32_t>(c >> 1) & 1u);
      const long long w1 = p.trace ? clock64() : 0;
      tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * kTile + h * 64 + c0), v);
#pragma unroll
        for (int i = 0; i < 16; ++i) accd[c0 + i] += (double)__uint_as_float(v[i]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(b ? te1 : te0);
      if (p.trace) {
        ew += w1 - w0;
        ef += clock64() - w1;
      }
    }
    if (p.trace && threadIdx.x == 64) {
      const long long sl = ((long long)blockIdx.y * gridDim.x + blockIdx.x) * 12;
      p.trace[sl + 8] = ew;
      p.trace[sl + 9] = ef;
    }
    double* S = reinterpret_cast<double*>(smem);   // [128][kEpiPitch]; this CTA's ring is idle
#pragma unroll
    for (int i = 0; i < 64; ++i) S[r * kEpiPitch + h * 64 + i] = accd[i];
    if (p.trace != nullptr && threadIdx.x == 64) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      const long long slot = ((long long)blockIdx.y * gridDim.x + blockIdx.x) * 12;
      p.trace[slot + 0] = t_start;
      p.trace[slot + 1] = t;
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      p.trace[slot + 3] = sm;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp >= 2) {
    const int n = p.ld / kTile;
    const bool write = (I < n) && (MODE == 2 || I <= J);
    mx_tile_epilogue<MODE, TF32>(reinterpret_cast<double*>(smem), I, J, job, blockIdx.x, write, p, red);
    if (p.trace != nullptr && threadIdx.x == 64) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      p.trace[((long long)blockIdx.y * gridDim.x + blockIdx.x) * 12 + 2] = t;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();                      // the pair leaves together (remote barriers, shared TMEM allocation)
  tc_fence_after();
  if (warp == 1) tmem_dealloc_cg2(tmem, 2 * kTile);
}

template <int MODE, bool TF32>
static cudaError_t launch_mx2_t(const CUtensorMap& tmP, const CUtensorMap& tmQ, const MxParams& p, int batch,
                                cudaStream_t st) {
  static unsigned long long attr = 0;
  smem_attr(ns_mx2_product_kernel<MODE, TF32>, kMx2SmemBytes, attr);
  dim3 grid(p.n_tiles, batch);   // n_tiles = 2 x pairs: one cluster of 2 per pair
  ns_mx2_product_kernel<MODE, TF32><<<grid, kMxThreads, kMx2SmemBytes, st>>>(tmP, tmQ, p);
  return cudaGetLastError();
}

cudaError_t launch_mx2_product(const CUtensorMap& tmP, const CUtensorMap& tmQ64, const MxParams& p, int batch,
                               cudaStream_t st) {
  if (p.tf32) {
    if (p.mode == 0) return launch_mx2_t<0, true>(tmP, tmQ64, p, batch, st);
    if (p.mode == 1) return launch_mx2_t<1, true>(tmP, tmQ64, p, batch, st);
    return launch_mx2_t<2, true>(tmP, tmQ64, p, batch, st);
  }
  if (p.mode == 0) return launch_mx2_t<0, false>(tmP, tmQ64, p, batch, st);
  if (p.mode == 1) return launch_mx2_t<1, false>(tmP, tmQ64, p, batch, st);
  return launch_mx2_t<2, false>(tmP, tmQ64, p, batch, st);
}

cudaError_t launch_split_planes(const double* X, void* planes, int d_pad, int batch, cudaStream_t st, bool tf32) {
  const long long n = (long long)d_pad * d_pad;
  long long blocks = (n * batch + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  if (tf32) ns_split_planes_kernel<true><<<(unsigned)blocks, 256, 0, st>>>(X, planes, n, batch);
  else ns_split_planes_kernel<false><<<(unsigned)blocks, 256, 0, st>>>(X, planes, n, batch);
  return cudaGetLastError();
}

template <int MODE, bool TF32>
static cudaError_t launch_mx_t(const CUtensorMap& tmP, const CUtensorMap& tmQ, const MxParams& p, int batch,
                               cudaStream_t st) {
  static unsigned long long attr = 0;
  smem_attr(ns_mx_product_kernel<MODE, TF32>, kMxSmemBytes, attr);
  dim3 grid(p.n_tiles, batch);
  ns_mx_product_kernel<MODE, TF32><<<grid, kMxThreads, kMxSmemBytes, st>>>(tmP, tmQ, p);
  return cudaGetLastError();
}

cudaError_t launch_mx_product(const CUtensorMap& tmP, const CUtensorMap& tmQ, const MxParams& p, int batch,
                              cudaStream_t st) {
  if (p.tf32) {
    if (p.mode == 0) return launch_mx_t<0, true>(tmP, tmQ, p, batch, st);
    if (p.mode == 1) return launch_mx_t<1, true>(tmP, tmQ, p, batch, st);
    return launch_mx_t<2, true>(tmP, tmQ, p, batch, st);
  }
  if (p.mode == 0) return launch_mx_t<0, false>(tmP, tmQ, p, batch, st);
  if (p.mode == 1) return launch_mx_t<1, false>(tmP, tmQ, p, batch, st);
  return launch_mx_t<2, false>(tmP, tmQ, p, batch, st);
}

}  // namespace nsr
