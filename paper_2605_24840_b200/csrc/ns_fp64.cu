// FP64 Newton–Schulz kernels for sm_100a (B200).
//
// Hot path (BASELINE north_star; eq:NS P:373-379, divide convention C1):
//   X_0 = (H - sI)/alpha                      ns_init_kernel        (HBM-bound, O(d^2))
//   Y_j = X_j X_j   + r_j = ||Y_j - I||_F      ns_product_kernel<0>  (symmetric: upper tiles only)
//   decide: rho_j < tol | j == max_steps       ns_decide_kernel      (1 CTA per problem)
//   X_{j+1} = 1.5 X_j - 0.5 X_j Y_j  + tr      ns_product_kernel<1>  (Z = X Y is symmetric since
//                                                                     X and Y commute)
//   R = X_steps                               ns_copy_out_kernel
//
// Contraction core: C_IJ = sum_k P[I,k] Q[J,k] for 128x128 output tiles with I <= J.
// Both operands are ROW panels of symmetric matrices (Y = X X^T, Z = X Y^T), so one
// TMA box shape serves both.  FP64 has no tcgen05 kind on sm_100a; the FP64 tensor
// instruction is warp-level DMMA (mma.sync m8n8k4 .f64, SASS DMMA.8x8x4), fed here by
// a TMA + mbarrier ring with a dedicated producer warp and 8 DMMA consumer warps.
// Shared-memory tiles use the TMA 128-byte swizzle; the consumer's k-permutation
// (k = 4t + s within a 16-wide slab) turns each fragment fetch into a conflict-free
// 128-bit LDS.  Epilogue: tile staged through shared memory, written row-major and
// mirrored (bitwise-symmetric output), with per-tile residual / trace partials that
// the decide kernel reduces in a fixed order (deterministic).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <type_traits>

#include "ns_internal.h"

#ifndef NS_K64_ROT0
#define NS_K64_ROT0 0   // 1: square launches rotate K the same way (measured: no gain, 3.53 vs 3.51 ms at cfg1)
#endif
#include "ns_ptx.cuh"

namespace nsr {

// --------------------------------------------------------------------------------------
// X_0 = (H - sI)/alpha from the UPPER triangle of H, zero-padded to d_pad.
// 64x64 blocks, 16 independent loads per thread in flight; block (bi,bj) reads H's tile (min,max)
// and writes its own tile (transposed through shared memory below the diagonal).
// --------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) ns_init_kernel(const double* __restrict__ H, long long ldh,
                                                      long long h_stride, double* __restrict__ X,
                                                      const JobParams* __restrict__ jobs, int d, int d_pad, int rb0) {
  __shared__ double t[64][65];
  const int job = blockIdx.z;
  const int bi = blockIdx.y + rb0, bj = blockIdx.x;
  const double* Hj = H + (long long)job * h_stride;
  double* Xj = X + (long long)job * d_pad * (long long)d_pad;
  const double s = jobs[job].s, alpha = jobs[job].alpha;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 64 x 4
  const int ri = min(bi, bj), rj = max(bi, bj);           // source tile in the upper triangle
  double v[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int gi = ri * 64 + ty + 4 * u, gj = rj * 64 + tx;
    v[u] = (gi < d && gj < d && gi <= gj) ? Hj[(long long)gi * ldh + gj] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < 16; ++u) t[ty + 4 * u][tx] = v[u];
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int gi = bi * 64 + ty + 4 * u, gj = bj * 64 + tx;
    double x = 0.0;
    if (gi < d && gj < d) {
      const double h = (gi <= gj) ? t[gi - ri * 64][gj - rj * 64] : t[gj - ri * 64][gi - rj * 64];
      x = (gi == gj) ? (h - s) / alpha : h / alpha;
    }
    Xj[(long long)gi * d_pad + gj] = x;
  }
}

// tr X per 128-row diagonal block (fixed-order block reduction) -> tr_partial[job*n + b].
__global__ void __launch_bounds__(128) ns_trace_partials_kernel(const double* __restrict__ X, int d, int d_pad,
                                                                double* __restrict__ tr_partial, int job_stride) {
  __shared__ double red[4];
  const int job = blockIdx.y, b = blockIdx.x, n = gridDim.x;
  const int i = b * kTile + threadIdx.x;
  double v = (i < d) ? X[(long long)job * d_pad * d_pad + (long long)i * d_pad + i] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) tr_partial[(long long)job * (job_stride > 0 ? job_stride : n) + b] = ((red[0] + red[1]) + red[2]) + red[3];
}

// --------------------------------------------------------------------------------------
// Symmetric-output product kernel (one 128x128 upper tile per CTA).
// --------------------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    ns_product_kernel(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmQ,
                      const ProdParams p) {
  int job = blockIdx.y;
  if (p.job_list != nullptr) {                          // batched: compacted list of active jobs
    if ((int)blockIdx.y >= *p.n_job_list) return;
    job = p.job_list[blockIdx.y];
  }
  if (p.state != nullptr && p.state[job].done) return;  // uniform per CTA

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  double* sA = reinterpret_cast<double*>(smem);                                           // [stages*kSPS][128*16]
  double* sB = reinterpret_cast<double*>(smem + kStages * kSPS * kTile * kBK * 8);       // [stages*kSPS][128*16]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  __shared__ double red[kConsumerWarps];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int2 tile = p.tiles[blockIdx.x];
  const int I = tile.x, J = tile.y;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // ---------------- TMA ring, driven by thread 0 between its own DMMA work ----------------
  // 8 warps only (2 per SMSP) so each thread may use up to 255 registers; thread 0 fills the first
  // kStages stages up front and, each time all warps have released a stage (empty barrier),
  // refills that slot with the stage kStages ahead.
  const int nst = p.nk / kSPS;
  auto issue = [&](int kt) {
    const int s = kt % kStages;
    mbar_arrive_expect_tx(&full[s], kStageBytes);
#pragma unroll
    for (int u = 0; u < kSPS; ++u) {
      tma_load_3d(sA + (s * kSPS + u) * kTile * kBK, &tmP, (kt * kSPS + u) * kBK, I * kTile, job, &full[s]);
      tma_load_3d(sB + (s * kSPS + u) * kTile * kBK, &tmQ, (kt * kSPS + u) * kBK, J * kTile, job, &full[s]);
    }
  };
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmP);
    tma_prefetch_desc(&tmQ);
    for (int kt = 0; kt < kStages && kt < nst; ++kt) issue(kt);
  }

  // ---------------- DMMA: warp tile 64 (rows of P) x 32 (rows of Q) ----------------
  const int cw = warp;            // 0..7
  const int wm = cw >> 2;         // 0..1  -> rows wm*64
  const int wn = cw & 3;          // 0..3  -> cols wn*32
  const int g = lane >> 2, t = lane & 3;
  // byte offsets inside a 128x16-double swizzled tile: row r -> r*128, 16-B chunk c -> (c ^ (r&7))*16;
  // r & 7 == g for every fragment row below.
  const uint32_t off_h0 = static_cast<uint32_t>(((2 * t + 0) ^ g) << 4);
  const uint32_t off_h1 = static_cast<uint32_t>(((2 * t + 1) ^ g) << 4);
  const uint32_t a_row = static_cast<uint32_t>((wm * 64 + g) * 128);
  const uint32_t b_row = static_cast<uint32_t>((wn * 32 + g) * 128);
  const uint32_t sA_u32 = smem_u32(sA), sB_u32 = smem_u32(sB);

  double acc[8][4][2];
#pragma unroll
  for (int mi = 0; mi < 8; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

  // MODE 1 reads the 128x128 tile of X_j in its epilogue: ask L2 for it a few stages before the end of
  // the k loop (at small d -- the batched configs -- that read was an exposed HBM latency per CTA)
  const int pf_kt = nst > 8 ? nst - 8 : 0;
  for (int kt = 0; kt < nst; ++kt) {
    const int s = kt % kStages;
    if (MODE == 1 && kt == pf_kt) {
      const double* Xt = p.Xold + (long long)job * p.job_stride + (long long)(I * kTile) * p.ld + J * kTile;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int l = threadIdx.x * 4 + u;     // 1024 lines of 128 B: row l >> 3, 16-double chunk l & 7
        prefetch_l2(Xt + (long long)(l >> 3) * p.ld + (l & 7) * 16);
      }
    }
    if (threadIdx.x == 0 && kt >= 1 && kt - 1 + kStages < nst) {
      // every warp released stage kt-1: refill its slot with stage kt-1+kStages
      const int sp = (kt - 1) % kStages;
      mbar_wait(&empty[sp], static_cast<uint32_t>((kt - 1) / kStages) & 1u);
      issue(kt - 1 + kStages);
    }
    mbar_wait(&full[s], static_cast<uint32_t>(kt / kStages) & 1u);
#pragma unroll
    for (int hh = 0; hh < 2 * kSPS; ++hh) {
      const int h = hh & 1;
      const uint32_t aS = sA_u32 + (s * kSPS + (hh >> 1)) * (kTile * kBK * 8) + a_row;
      const uint32_t bS = sB_u32 + (s * kSPS + (hh >> 1)) * (kTile * kBK * 8) + b_row;
      const uint32_t off = h ? off_h1 : off_h0;
      // all fragments of this half-slab first, then the DMMAs k-step-major: the two updates of an
      // accumulator are 32 DMMAs apart
      double a[8][2], b[4][2];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) lds128(bS + ni * 8 * 128 + off, b[ni][0], b[ni][1]);
#pragma unroll
      for (int mi = 0; mi < 8; ++mi) lds128(aS + mi * 8 * 128 + off, a[mi][0], a[mi][1]);
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int mi = 0; mi < 8; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi][e], b[ni][e]);
    }
    fence_proxy_async();                 // generic reads of the slot before the TMA refill (see 64-tile kernel)
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // ---------------- epilogue ----------------
  // All stages consumed by every consumer warp before the ring is reused as staging.
  named_bar_sync(1, 32 * kConsumerWarps);
  double* S = reinterpret_cast<double*>(smem);   // [128][kEpiPitch]
#pragma unroll
  for (int mi = 0; mi < 8; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int r = wm * 64 + mi * 8 + g;
      const int c = wn * 32 + ni * 8 + 2 * t;
      S[r * kEpiPitch + c] = acc[mi][ni][0];
      S[r * kEpiPitch + c + 1] = acc[mi][ni][1];
    }
  named_bar_sync(1, 32 * kConsumerWarps);

  const int tid = threadIdx.x;        // 0..255
  const long long ld = p.ld;
  const long long base = (long long)job * p.job_stride;
  double* C = p.C + base;
  const bool diag = (I == J);
  double part = 0.0;

  if (MODE == 2) {
    // dense product tile, no symmetry assumed: C_IJ only
    for (int idx = tid; idx < kTile * kTile; idx += 256) {
      const int r = idx >> 7, c = idx & 127;
      C[(long long)(I * kTile + r) * ld + J * kTile + c] = S[r * kEpiPitch + c];
    }
  } else if (MODE == 0) {
    // Y tile + residual partial: off-diagonal tiles count twice (Y_JI = Y_IJ^T).
    if (!diag) {
      for (int idx = tid; idx < kTile * kTile; idx += 256) {
        const int r = idx >> 7, c = idx & 127;
        const double v = S[r * kEpiPitch + c];
        C[(long long)(I * kTile + r) * ld + J * kTile + c] = v;
        part += v * v;
      }
      part *= 2.0;
      for (int idx = tid; idx < kTile * kTile; idx += 256) {
        const int r = idx >> 7, c = idx & 127;   // mirror row J*128+r, col I*128+c  <- tile (c, r)
        C[(long long)(J * kTile + r) * ld + I * kTile + c] = S[c * kEpiPitch + r];
      }
    } else {
      for (int idx = tid; idx < kTile * kTile; idx += 256) {
        const int r = idx >> 7, c = idx & 127;
        const double v = (r <= c) ? S[r * kEpiPitch + c] : S[c * kEpiPitch + r];
        C[(long long)(I * kTile + r) * ld + I * kTile + c] = v;
        if (r < c) {
          part += 2.0 * v * v;
        } else if (r == c) {
          const double e = (I * kTile + r < p.d) ? v - 1.0 : v;
          part += e * e;
        }
      }
    }
  } else {
    // X_{j+1} = 1.5 X_j - 0.5 Z,  Z = X_j Y_j ; trace partial on diagonal tiles.
    const double* X = p.Xold + base;
    if (!diag) {
      // X_j is read 8 elements at a time before any store (C may alias X as far as the compiler knows,
      // so a load per iteration would otherwise wait out a full memory latency: ~35% of a configs[1]
      // update launch in the ncu source view)
      for (int idx0 = tid; idx0 < kTile * kTile; idx0 += 8 * 256) {
        double xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int idx = idx0 + u * 256, r = idx >> 7, c = idx & 127;
          xv[u] = X[(long long)(I * kTile + r) * ld + J * kTile + c];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int idx = idx0 + u * 256, r = idx >> 7, c = idx & 127;
          const long long gidx = (long long)(I * kTile + r) * ld + J * kTile + c;
          const double v = fma(p.cb, S[r * kEpiPitch + c], p.ca * xv[u]);
          C[gidx] = v;
          S[r * kEpiPitch + c] = v;
        }
      }
      named_bar_sync(1, 32 * kConsumerWarps);
      for (int idx = tid; idx < kTile * kTile; idx += 256) {
        const int r = idx >> 7, c = idx & 127;
        C[(long long)(J * kTile + r) * ld + I * kTile + c] = S[c * kEpiPitch + r];
      }
    } else {
      for (int idx0 = tid; idx0 < kTile * kTile; idx0 += 8 * 256) {
        double xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int idx = idx0 + u * 256, r = idx >> 7, c = idx & 127;
          xv[u] = (r <= c) ? X[(long long)(I * kTile + r) * ld + I * kTile + c] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int idx = idx0 + u * 256, r = idx >> 7, c = idx & 127;
          if (r <= c) {
            double v = fma(p.cb, S[r * kEpiPitch + c], p.ca * xv[u]);
            if (r == c && I * kTile + r < p.d) {
              v += p.cc;
              part += v;
            }
            S[r * kEpiPitch + c] = v;
          }
        }
      }
      named_bar_sync(1, 32 * kConsumerWarps);
      for (int idx = tid; idx < kTile * kTile; idx += 256) {
        const int r = idx >> 7, c = idx & 127;
        C[(long long)(I * kTile + r) * ld + I * kTile + c] = (r <= c) ? S[r * kEpiPitch + c] : S[c * kEpiPitch + r];
      }
    }
  }

  if (MODE == 2) return;
  if (p.n_dst > 0) {
    // peer-memory exchange: the same tile (and, if remote_mirror, its mirror) into every other destination;
    // S holds the final values (MODE 1 updated it in place; diagonal tiles are valid on and above the diagonal)
    named_bar_sync(1, 32 * kConsumerWarps);
    for (int q = 0; q < p.n_dst; ++q) {
      double* Cq = p.dst[q] + base;
      if (Cq == C) continue;
      if (!diag) {
        for (int idx = tid; idx < kTile * kTile; idx += 256) {
          const int r = idx >> 7, c = idx & 127;
          Cq[(long long)(I * kTile + r) * ld + J * kTile + c] = S[r * kEpiPitch + c];
        }
        if (p.remote_mirror)   // else the receiver mirrors its peers' off-diagonal tiles after the barrier
          for (int idx = tid; idx < kTile * kTile; idx += 256) {
            const int r = idx >> 7, c = idx & 127;
            Cq[(long long)(J * kTile + r) * ld + I * kTile + c] = S[c * kEpiPitch + r];
          }
      } else {
        for (int idx = tid; idx < kTile * kTile; idx += 256) {
          const int r = idx >> 7, c = idx & 127;
          Cq[(long long)(I * kTile + r) * ld + I * kTile + c] = (r <= c) ? S[r * kEpiPitch + c] : S[c * kEpiPitch + r];
        }
      }
    }
    __threadfence_system();                // this thread's remote stores performed before the CTA retires
  }
  // fixed-order reduction of `part` over the 256 consumer threads
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) red[cw] = part;
  named_bar_sync(1, 32 * kConsumerWarps);
  if (tid == 0) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w) s += red[w];
    if (p.n_dst > 0) {
      const long long gt = (long long)p.gt_off + (long long)blockIdx.x * p.gt_stride;
      for (int q = 0; q < p.n_dst; ++q) {
        if (MODE == 0) p.dst_part[q][(long long)job * p.n_tiles_total + gt] = s;
        else if (diag) p.dst_part[q][(long long)job * (p.ld / kTile) + I] = s;
      }
      __threadfence_system();
    } else if (MODE == 0) {
      p.partial[(long long)job * p.n_tiles + (p.part_slot ? p.part_slot[blockIdx.x] : (int)blockIdx.x)] = s;
    } else if (diag) {
      p.partial[(long long)job * (p.ld / kTile) + I] = s;
    }
  }
}

// --------------------------------------------------------------------------------------
// 64x64-tile variant for small and batched problems (d_pad <= 1024): the upper triangle in 64-tiles
// wastes less on diagonal tiles (d = 256: 10 tiles of 64^2 instead of 3 of 128^2 per product, 17%
// fewer MACs), gives 4x more CTAs to a single mid-size problem, and with 96 KB of shared memory and
// 128 threads two CTAs share an SM, so one CTA's epilogue overlaps the other's DMMA loop.
// Same scheme as ns_product_kernel: TMA ring (box 16 x 64, 128-B swizzle), thread 0 refills, 4 DMMA
// warps with 32x32 warp tiles and the k-permuted conflict-free LDS.128 fragments, staged epilogue.
// --------------------------------------------------------------------------------------
__device__ __forceinline__ void stg_v2(double* p, double x, double y) {
  asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(x), "d"(y) : "memory");
}
#ifndef NS_K64_HH_UNROLL
#define NS_K64_HH_UNROLL 4   // half-slabs of a ring stage unrolled in the K loop (4 = the whole stage)
#endif
constexpr int kHHUnroll = NS_K64_HH_UNROLL;
#ifndef NS_K64_MIRROR8
#define NS_K64_MIRROR8 1   // 0: mirror by one 16-byte store after a lane shuffle (8 rows x 64 B per warp store)
#endif
#ifndef NS_P64_TRACE
#define NS_P64_TRACE 0   // 1: every CTA of the 64-tile kernel records %globaltimer phase stamps (tools/p64_trace.py)
#endif
#if NS_P64_TRACE
// g_p64_trace[0] = record counter; record r at 1 + 10 r: smid | mode << 16 | diag << 17, start, first stage
// landed, end, job << 32 | tile, K loop done of warps 0..3, 0
__device__ unsigned long long* g_p64_trace = nullptr;
__device__ unsigned long long g_p64_cap = 0;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif
template <int MODE>
__global__ void __launch_bounds__(k64Threads, k64MinBlocks)
    ns_product64_kernel(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmQ,
                        const ProdParams p) {
  int job = blockIdx.y;
  if (p.job_list != nullptr) {
    if ((int)blockIdx.y >= *p.n_job_list) return;
    job = p.job_list[blockIdx.y];
  }
  // the compacted list holds only running jobs (ns_compact_kernel after the last decide): no state read
  else if (p.state != nullptr && p.state[job].done) return;
#if NS_P64_TRACE
  unsigned long long tr_t0 = gtimer(), tr_t1 = 0;
  __shared__ unsigned long long tr_wend[k64Threads / 32], tr_wst[k64Threads / 32];
#endif
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  double* sA = reinterpret_cast<double*>(smem);                                      // [stages*k64SPS][64*16]
  double* sB = reinterpret_cast<double*>(smem + k64Stages * k64SPS * k64Tile * kBK * 8);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + k64Stages * k64StageBytes);
  uint64_t* empty = full + k64Stages;
  __shared__ double red[k64Threads / 32];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int2 tile = p.tiles[blockIdx.x];
  const int I = tile.x, J = tile.y;        // 64-blocks
  if (threadIdx.x == 0) {
    for (int s = 0; s < k64Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], k64Threads / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int nst = p.nk / k64SPS;
  // MODE 1 walks K starting after the tile's own column block J (stage units 2J, 2J+1 of 32 columns
  // come last), so when the loop ends the ring still holds X_j[I rows][J columns] -- the tile the
  // update epilogue needs -- and no global re-read of X_j is required.
  constexpr int kJS = 4 / k64SPS;         // stages per 64-column block
  const int koff = (MODE == 1 || NS_K64_ROT0) ? (kJS * J + kJS) % nst : 0;
  // a diagonal tile of a square (P == Q) needs one row panel, not two: the B fragments come from sA
  const bool share = (MODE == 0) && (I == J) && p.diag_tri && p.same_pq;
  auto issue = [&](int kt) {
    const int s = kt % k64Stages;
    const int kb = (kt + koff) % nst;
    mbar_arrive_expect_tx(&full[s], share ? k64StageBytes / 2 : k64StageBytes);
#pragma unroll
    for (int u = 0; u < k64SPS; ++u) {
      tma_load_3d(sA + (s * k64SPS + u) * k64Tile * kBK, &tmP, (kb * k64SPS + u) * kBK, I * k64Tile, job, &full[s]);
      if (!share)
        tma_load_3d(sB + (s * k64SPS + u) * k64Tile * kBK, &tmQ, (kb * k64SPS + u) * kBK, J * k64Tile, job, &full[s]);
    }
  };
  // X_j(r, c..c+1) of this tile (c even) from the ring after the K loop: the block's 16-column slab q sits in
  // the slot of stage nst - kJS + q / k64SPS; 128-B swizzle (16-B chunk of row r at chunk ^ (r & 7))
  // (a ring shallower than the block, k64Stages * k64SPS < 4, has overwritten its first slabs: those come from
  // L2 instead)
  auto x_ring = [&](int r, int c) -> double2 {
    const int q = c >> 4;                        // 16-column slab of the block
    if (k64Stages * k64SPS < 4 && q < 4 - k64Stages * k64SPS)
      return *reinterpret_cast<const double2*>(p.Xold + (long long)job * p.job_stride +
                                               (long long)(I * k64Tile + r) * p.ld + J * k64Tile + c);
    const int slot = (nst - kJS + q / k64SPS) % k64Stages;
    const int cs = c & 15;
    const double* slab = sA + (slot * k64SPS + q % k64SPS) * (k64Tile * kBK);
    return *reinterpret_cast<const double2*>(slab + r * kBK + (((cs >> 1) ^ (r & 7)) << 1));
  };
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmP);
    tma_prefetch_desc(&tmQ);
    for (int kt = 0; kt < k64Stages && kt < nst; ++kt) issue(kt);
  }
  constexpr int NWP = k64Threads / 32;        // DMMA warps per CTA: 4 (32x32 warp tiles) or 8 (32x16)
  constexpr int WN = 64 / (NWP / 2);          // warp tile columns
  constexpr int NI = WN / 8;                  // 8-column fragments per warp
  const int wm = warp / (NWP / 2), wn = warp % (NWP / 2);   // warp tile rows wm*32, cols wn*WN
  const int g = lane >> 2, t = lane & 3;
  const uint32_t off_h0 = static_cast<uint32_t>(((2 * t + 0) ^ g) << 4);
  const uint32_t off_h1 = static_cast<uint32_t>(((2 * t + 1) ^ g) << 4);
  const uint32_t sA_u32 = smem_u32(sA), sB_u32 = smem_u32(sB);
  const bool diag = (I == J);
  // K loop: ring bookkeeping around a per-warp compute step on stage s
  auto mainloop = [&](auto&& compute) {
    for (int kt = 0; kt < nst; ++kt) {
      const int s = kt % k64Stages;
      if (threadIdx.x == 0 && kt >= 1 && kt - 1 + k64Stages < nst) {
        const int sp = (kt - 1) % k64Stages;
        mbar_wait(&empty[sp], static_cast<uint32_t>((kt - 1) / k64Stages) & 1u);
        issue(kt - 1 + k64Stages);
      }
      mbar_wait(&full[s], static_cast<uint32_t>(kt / k64Stages) & 1u);
#if NS_P64_TRACE
      if (kt == 0 && threadIdx.x == 0) tr_t1 = gtimer();
#endif
      compute(s);
      // the slot is refilled by TMA (async proxy) once every warp has released it: order this warp's generic-
      // proxy reads of it before the release (without the fence, 3 CTAs/SM with a 2-stage ring produced
      // nondeterministic results -- a refill overtaking the last LDS of the slot)
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  };
  // ---------------- epilogue straight from the accumulator registers ----------------
  // Lane (g, t) of a fragment holds C[r][c], C[r][c+1] (r = 8-row base + g, c = 8-col base + 2t): one 16-byte
  // store for the tile (8 rows x 64 contiguous bytes per warp store) and two 8-byte stores for the mirror,
  // C[c][r] and C[c+1][r] (4 rows x 64 bytes each; NS_K64_MIRROR8=0: one 16-byte store after a shuffle with lane
  // g ^ 1 -- even g takes row c: (r, r+1), odd g row c+1: (r-1, r)).  No
  // shared-memory staging and no block barrier before the stores (the staged epilogue -- fragments to a padded
  // smem tile, then coalesced row and column passes -- took ~25% of a CTA's warp time in ncu; cfg1 118.3 ->
  // 115.9 ms).  Diagonal 8x8 blocks keep c >= r and mirror it, so every stored matrix is bitwise symmetric.
  const long long ld = p.ld;
  const long long base = (long long)job * p.job_stride;
  double* C = p.C + base;
  const int i0 = I * k64Tile, j0 = J * k64Tile;
  double part = 0.0;
  unsigned dbg_x = 0;
  auto dbg_epilogue = [&]() {   // sensitivity experiments: idle time vs issued instructions in a CTA's epilogue
    if (p.dbg_sleep > 0) __nanosleep(p.dbg_sleep);
    if (p.dbg_int) {
      unsigned x0 = lane, x1 = 7, x2 = 9, x3 = 11;
      for (int i = 0; i < p.dbg_int; ++i) {
        asm volatile("lop3.b32 %0, %0, %1, 0x5a5a5a5a, 0x96;" : "+r"(x0) : "r"(x1));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(x1) : "r"(x2));
        asm volatile("lop3.b32 %0, %0, %1, 0x33333333, 0x96;" : "+r"(x2) : "r"(x3));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(x3) : "r"(x0));
      }
      dbg_x = x0 + x1 + x2 + x3;
    }
  };
  // MODE 0: off-diagonal squares in four independent DFMA chains (weight 2 applied once at the end): the FP64
  // pipe is busy with the other CTAs' DMMAs, so the epilogue issues as few, and as independent, FP64
  // instructions as it can
  double sq0 = 0.0, sq1 = 0.0, sq2 = 0.0, sq3 = 0.0;
  const bool godd = (g & 1) != 0;
  // off-diagonal 8x8 block (r in rows, c >= every r): tile store + mirror, MODE 0 residual weight 2
  // tp = &C[r][c] and mp = this lane's mirror address (even g: &C[c][r], odd g: &C[c+1][r-1]) are formed by the
  // callers from per-warp base pointers with constant strides: next to a saturated DMMA stream every issued
  // integer instruction costs ~0.5 clk of DMMA time (profiles/r02_dmma_issue.txt), and the per-fragment 64-bit
  // address arithmetic was most of this epilogue's ~45 instructions per fragment
  const long long ld8 = 8 * ld;
  constexpr int kGo = NS_K64_MIRROR8 ? 0 : 1;   // 16-byte mirror stores: odd g stores row c + 1 from column r - 1
  auto put_full = [&](double* tp, double* mp, double v0, double v1, int ch) {
    if (MODE == 0) {
      if (ch & 1) {
        sq2 = fma(v0, v0, sq2);
        sq3 = fma(v1, v1, sq3);
      } else {
        sq0 = fma(v0, v0, sq0);
        sq1 = fma(v1, v1, sq1);
      }
    }
    stg_v2(tp, v0, v1);
#if NS_K64_MIRROR8
    // mirror by two 8-byte stores (C[c][r] and C[c+1][r]; a warp store covers 4 rows x 64 contiguous bytes): no
    // shuffle and no lane-parity selects -- 3 instead of 10 instructions per fragment next to the DMMA stream
    mp[0] = v0;
    mp[ld] = v1;
#else
    const double send = godd ? v0 : v1;
    const double recv = __shfl_xor_sync(0xffffffffu, send, 4);
    stg_v2(mp, godd ? recv : v0, godd ? v1 : recv);
#endif
  };
  // 8x8 block on the diagonal of a diagonal tile: elements c >= r (+ mirror), identity / trace / + cc I on c == r
  auto put_diag = [&](int r, int c, double v0, double v1) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int cc = c + h;
      double v = h ? v1 : v0;
      if (cc < r) continue;
      if (cc == r) {
        const bool in = i0 + r < p.d;
        if (MODE == 0) {
          const double e = in ? v - 1.0 : v;
          part = fma(e, e, part);
        } else if (in) {
          v += p.cc;
          part += v;
        }
      } else if (MODE == 0) {
        if (h) sq1 = fma(v, v, sq1);
        else sq0 = fma(v, v, sq0);
      }
      C[(long long)(i0 + r) * ld + i0 + cc] = v;
      if (cc != r) C[(long long)(i0 + cc) * ld + i0 + r] = v;
    }
  };
  if (!diag || !p.diag_tri) {
    const uint32_t a_row = static_cast<uint32_t>((wm * 32 + g) * 128);
    const uint32_t b_row = static_cast<uint32_t>((wn * WN + g) * 128);
    double acc[4][NI][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
    mainloop([&](int s) {
#pragma unroll(kHHUnroll)
      for (int hh = 0; hh < 2 * k64SPS; ++hh) {
        const int h = hh & 1;
        const uint32_t aS = sA_u32 + (s * k64SPS + (hh >> 1)) * (k64Tile * kBK * 8) + a_row;
        const uint32_t bS = sB_u32 + (s * k64SPS + (hh >> 1)) * (k64Tile * kBK * 8) + b_row;
        const uint32_t off = h ? off_h1 : off_h0;
        double a[4][2], b[NI][2];
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) lds128(bS + ni * 8 * 128 + off, b[ni][0], b[ni][1]);
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) lds128(aS + mi * 8 * 128 + off, a[mi][0], a[mi][1]);
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi][e], b[ni][e]);
      }
    });
    dbg_epilogue();
    if (p.dbg_sleep < 0) {   // timing only: no epilogue at all (one store keeps the accumulators live)
      double sum = 0.0;
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) sum += acc[mi][ni][0] + acc[mi][ni][1];
      if (sum == 1.2345e300) C[0] = sum;
      return;
    }
    if (MODE == 1) {   // X_{j+1} = ca X_j + cb Z in registers, X_j from the ring
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          const double2 x = x_ring(wm * 32 + mi * 8 + g, wn * WN + ni * 8 + 2 * t);
          acc[mi][ni][0] = fma(p.cb, acc[mi][ni][0], p.ca * x.x);
          acc[mi][ni][1] = fma(p.cb, acc[mi][ni][1], p.ca * x.y);
        }
    }
#if NS_P64_TRACE
    if (lane == 0) tr_wend[warp] = gtimer();
#endif
    double* const T0 = C + (long long)(i0 + wm * 32 + g) * ld + j0 + wn * WN + 2 * t;
    double* const M0 = C + (long long)(j0 + wn * WN + 2 * t + kGo * (godd ? 1 : 0)) * ld + i0 + wm * 32 + g - kGo * (godd ? 1 : 0);
    if (!diag) {
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
          put_full(T0 + mi * ld8 + ni * 8, M0 + ni * ld8 + mi * 8, acc[mi][ni][0], acc[mi][ni][1], mi * NI + ni);
    } else {   // full diagonal tile (NS_DIAG_TRI=0 only): upper 8x8 blocks + the blocks on the diagonal
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          const int rb = wm * 4 + mi, cb = wn * NI + ni;   // 8-blocks (warp-uniform)
          if (rb < cb)
            put_full(T0 + mi * ld8 + ni * 8, M0 + ni * ld8 + mi * 8, acc[mi][ni][0], acc[mi][ni][1], ni);
          else if (rb == cb)
            put_diag(wm * 32 + mi * 8 + g, wn * WN + ni * 8 + 2 * t, acc[mi][ni][0], acc[mi][ni][1]);
        }
    }
  } else {
    // Diagonal tile: only the 36 upper-triangle 8x8 blocks (rb <= cb) of the 8x8 block grid are needed.
    // Each SM sub-partition (warps w, w + 4 when NWP = 8) takes block rows P and 7 - P: (8 - P) + (P + 1) = 9
    // blocks, so the four sub-partitions stay balanced (32x32 warp quadrants would leave one warp idle and one
    // at full load).  Batched d = 256: 17% fewer DMMAs per product.  NWP = 4: one warp per pair of rows;
    // NWP = 8: warp P takes row P, warp P + 4 row 7 - P.
    auto rows_warp = [&](auto WC, auto SC) {
      constexpr int W = decltype(WC)::value;
      constexpr bool SHARE = decltype(SC)::value;   // B fragments from sA; the A fragments are B fragments
      constexpr int P = W % 4;
      constexpr bool TWO = (NWP == 4);
      constexpr int R0 = (NWP == 8 && W >= 4) ? 7 - P : P, N0 = 8 - R0;
      constexpr int R1 = 7 - P, N1 = TWO ? P + 1 : 0;
      double c0[N0][2], c1[N1 > 0 ? N1 : 1][2];
#pragma unroll
      for (int i = 0; i < N0; ++i) c0[i][0] = c0[i][1] = 0.0;
#pragma unroll
      for (int i = 0; i < N1; ++i) c1[i][0] = c1[i][1] = 0.0;
      mainloop([&](int s) {
#pragma unroll(kHHUnroll)
        for (int hh = 0; hh < 2 * k64SPS; ++hh) {
          const int h = hh & 1;
          const uint32_t aS = sA_u32 + (s * k64SPS + (hh >> 1)) * (k64Tile * kBK * 8) + g * 128;
          const uint32_t bS = SHARE ? aS : sB_u32 + (s * k64SPS + (hh >> 1)) * (k64Tile * kBK * 8) + g * 128;
          const uint32_t off = h ? off_h1 : off_h0;
          constexpr int B0 = TWO ? (R0 < R1 ? R0 : R1) : R0;   // first B block needed
          double a0[2], a1[2], b[8][2];
#pragma unroll
          for (int cb = B0; cb < 8; ++cb) lds128(bS + cb * 8 * 128 + off, b[cb][0], b[cb][1]);
          if (SHARE) {   // same panel, same k-permutation: row block R's A fragment is its B fragment
            a0[0] = b[R0][0];
            a0[1] = b[R0][1];
            if (TWO) {
              a1[0] = b[R1][0];
              a1[1] = b[R1][1];
            }
          } else {
            lds128(aS + R0 * 8 * 128 + off, a0[0], a0[1]);
            if (TWO) lds128(aS + R1 * 8 * 128 + off, a1[0], a1[1]);
          }
#pragma unroll
          for (int e = 0; e < 2; ++e) {
#pragma unroll
            for (int i = 0; i < N0; ++i) dmma_8x8x4(c0[i][0], c0[i][1], a0[e], b[R0 + i][e]);
#pragma unroll
            for (int i = 0; i < N1; ++i) dmma_8x8x4(c1[i][0], c1[i][1], a1[e], b[R1 + i][e]);
          }
        }
      });
      if (MODE == 1) {
#pragma unroll
        for (int i = 0; i < N0; ++i) {
          const double2 x = x_ring(R0 * 8 + g, (R0 + i) * 8 + 2 * t);
          c0[i][0] = fma(p.cb, c0[i][0], p.ca * x.x);
          c0[i][1] = fma(p.cb, c0[i][1], p.ca * x.y);
        }
#pragma unroll
        for (int i = 0; i < N1; ++i) {
          const double2 x = x_ring(R1 * 8 + g, (R1 + i) * 8 + 2 * t);
          c1[i][0] = fma(p.cb, c1[i][0], p.ca * x.x);
          c1[i][1] = fma(p.cb, c1[i][1], p.ca * x.y);
        }
      }
#if NS_P64_TRACE
      if (lane == 0) tr_wend[warp] = gtimer();
#endif
      // block row R: fragment i is the 8x8 block (R, R + i) of this diagonal tile
      double* const TR0 = C + (long long)(i0 + R0 * 8 + g) * ld + i0 + R0 * 8 + 2 * t;
      double* const MR0 = C + (long long)(i0 + R0 * 8 + 2 * t + kGo * (godd ? 1 : 0)) * ld + i0 + R0 * 8 + g - kGo * (godd ? 1 : 0);
#pragma unroll
      for (int i = 0; i < N0; ++i) {
        if (i == 0) put_diag(R0 * 8 + g, R0 * 8 + 2 * t, c0[i][0], c0[i][1]);
        else put_full(TR0 + i * 8, MR0 + i * ld8, c0[i][0], c0[i][1], i);
      }
      double* const TR1 = C + (long long)(i0 + R1 * 8 + g) * ld + i0 + R1 * 8 + 2 * t;
      double* const MR1 = C + (long long)(i0 + R1 * 8 + 2 * t + kGo * (godd ? 1 : 0)) * ld + i0 + R1 * 8 + g - kGo * (godd ? 1 : 0);
#pragma unroll
      for (int i = 0; i < N1; ++i) {
        if (i == 0) put_diag(R1 * 8 + g, R1 * 8 + 2 * t, c1[i][0], c1[i][1]);
        else put_full(TR1 + i * 8, MR1 + i * ld8, c1[i][0], c1[i][1], i + 1);
      }
    };
    auto rows_any = [&](auto SC) {
      switch (warp) {
        case 0: rows_warp(std::integral_constant<int, 0>{}, SC); break;
        case 1: rows_warp(std::integral_constant<int, 1>{}, SC); break;
        case 2: rows_warp(std::integral_constant<int, 2>{}, SC); break;
        case 3: rows_warp(std::integral_constant<int, 3>{}, SC); break;
#if NS_K64_WARPS == 8
        case 4: rows_warp(std::integral_constant<int, 4>{}, SC); break;
        case 5: rows_warp(std::integral_constant<int, 5>{}, SC); break;
        case 6: rows_warp(std::integral_constant<int, 6>{}, SC); break;
        default: rows_warp(std::integral_constant<int, 7>{}, SC); break;
#endif
      }
    };
    if (MODE == 0 && share) rows_any(std::true_type{});
    else rows_any(std::false_type{});
  }
  const int tid = threadIdx.x;
#if NS_P64_TRACE
  if (lane == 0) tr_wst[warp] = gtimer();
#endif
  if (MODE == 0) part = fma(2.0, (sq0 + sq1) + (sq2 + sq3), part);
  if (dbg_x == 0x12345678u) part += 1.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) red[warp] = part;
  __syncthreads();
  if (tid == 0) {
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < k64Threads / 32; ++w) sum += red[w];
    if (MODE == 0) p.partial[(long long)job * p.n_tiles + (p.part_slot ? p.part_slot[blockIdx.x] : (int)blockIdx.x)] = sum;
    else if (diag) p.partial[(long long)job * (p.ld / k64Tile) + I] = sum;
#if NS_P64_TRACE
    if (g_p64_trace != nullptr) {
      const unsigned long long r = atomicAdd(g_p64_trace, 1ull);
      if (r < g_p64_cap) {
        unsigned long long* rec = g_p64_trace + 1 + 10 * r;
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        rec[0] = smid | ((unsigned long long)MODE << 16) | ((unsigned long long)diag << 17);
        rec[1] = tr_t0;
        rec[2] = tr_t1;
        rec[3] = gtimer();
        rec[4] = ((unsigned long long)job << 32) | blockIdx.x;
#pragma unroll
        for (int w = 0; w < 4; ++w) rec[5 + w] = tr_wend[w];
        unsigned long long wst = 0;
        for (int w = 0; w < 4; ++w) wst = tr_wst[w] > wst ? tr_wst[w] : wst;
        rec[9] = wst;   // last warp's stores issued
      }
    }
#endif
  }
}

// --------------------------------------------------------------------------------------
// Stop decision for step j (one CTA per problem); fixed-order reductions.
// --------------------------------------------------------------------------------------
__device__ __forceinline__ double block_sum_fixed(const double* v, int n, double* red) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += v[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  double tot = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
  return tot;
}

__global__ void __launch_bounds__(256) ns_decide_kernel(DevState* __restrict__ state, const JobParams* __restrict__ jobs,
                                                        const double* __restrict__ res_partial, int n_tiles,
                                                        const double* __restrict__ tr_partial, int n_diag,
                                                        LoopParams lp, int* n_active,
                                                        const double* __restrict__ res_ranks, int nranks) {
  __shared__ double red[8];
  const int job = blockIdx.x;
  DevState* st = state + job;
  if (st->done) return;
  if (lp.lowprec && st->sw) return;   // low-precision phase already left (look-ahead launch)
  double r2 = block_sum_fixed(res_partial + (long long)job * n_tiles, n_tiles, red);
  const double tr = block_sum_fixed(tr_partial + (long long)job * n_diag, n_diag, red);
  if (threadIdx.x != 0) return;
  if (res_ranks != nullptr) {   // sharded: per-rank sums gathered over NCCL, summed in rank order
    r2 = 0.0;
    for (int q = 0; q < nranks; ++q) r2 += res_ranks[q];
  }
  const double r = sqrt(r2);
  int flags = st->flags;
  int done = 0;
  const double sqd = sqrt((double)lp.d);
  if (!isfinite(r)) {
    flags |= 16;  // NS_F_NONFINITE
    done = 1;
  } else {
    // NS_F_SCALING_SUSPECT: a residual rise beyond the arithmetic's noise floor (FP64: 1e-10 sqrt(d);
    // BF16x3 phase of the mixed path: 1e-4 sqrt(d), the split-precision floor).
    const double slack = (lp.lowprec ? 1e-4 : 1e-10) * sqd;
    if (st->j > 0 && r > st->r_prev * (1.0 + 1e-12) + slack) flags |= 8;
    const double rho = lp.tol_mode ? r / sqd : r;
    if (lp.lowprec && st->j_small < 0 && r / sqd < lp.switch_tol) st->j_small = st->j;
    if (rho < lp.tol) {
      flags |= 1;  // NS_F_CONVERGED
      done = 1;
    } else if (st->j >= lp.max_steps) {
      flags |= 2;  // NS_F_MAX_STEPS
      done = 1;
    } else if (lp.lowprec && !st->sw &&
               (lp.switch_at >= 0 ? st->j >= lp.switch_at : r / sqd < lp.switch_tol)) {
      // mixed path: leave the low-precision phase at this j (re-anchor + FP64 from here, C16)
      st->sw = 1;
      st->sw_step = st->j;
      st->sw_residual = r;
      st->r_prev = INFINITY;   // the FP64 phase's first residual is not compared with a BF16x3 one
      st->residual = r;
      st->trace = tr;
      st->flags = flags;
      if (n_active) atomicSub(n_active, 1);
      return;
    }
  }
  st->residual = r;
  st->trace = tr;
  if (done) {
    const double half = ((double)lp.d - tr) * 0.5;
    long long cert = -1;                                   // no certificate for a non-finite iterate
    if (!(flags & 16) && isfinite(half)) {
      cert = (long long)floor(fabs(half) + 0.5);
      if (half < 0) cert = -cert;
      if (fabs(half - (double)cert) > 0.25) flags |= 32;  // NS_F_SHIFT_ON_SPECTRUM
    }
    if (cert != (long long)jobs[job].k) flags |= 4;       // NS_F_INDEX_MISMATCH
    st->cert = cert;
    st->flags = flags;
    st->done = 1;
    if (n_active) atomicSub(n_active, 1);
  } else {
    st->flags = flags;
    st->r_prev = r;
    // X_{j+1} will be returned if it is the max_steps iterate, or if its residual is certain to pass:
    // per eigenvalue e' = (1 - x'^2) = e^2 (3 + e)/4 <= e^2 for e = 1 - x^2 in [0, 1], so
    // r_{j+1} <= r_j^2 (half of the tolerance kept as margin for the products' rounding)
    const double tol_abs = lp.tol_mode ? lp.tol * sqd : lp.tol;
    if (st->j + 1 == lp.max_steps || (!lp.lowprec && r * r < 0.5 * tol_abs)) st->spec = st->j + 1;
    st->j += 1;
  }
}

__global__ void ns_zero_state_kernel(DevState* state, int batch, int* n_active) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < batch) {
    DevState z{};
    z.j_small = -1;
    z.sw_step = -1;
    state[i] = z;
  }
  if (i == 0 && n_active) *n_active = batch;
}

// R = X_{steps}: buffer chosen on device from state.j (ping-pong parity).
// R_job (d x d, leading dimension ldr) <- the returned iterate, 8 independent elements (or double2
// pairs when rows are 16-B aligned) per thread in flight over the flattened d*d range.
template <bool V2>
__global__ void __launch_bounds__(256) ns_copy_out_kernel(const double* __restrict__ Xa, const double* __restrict__ Xb,
                                                          int d, int d_pad, const DevState* __restrict__ state,
                                                          double* __restrict__ R, long long ldr, long long r_stride,
                                                          int row0, int rows) {
  const int job = blockIdx.y;
  const double* X = ((state[job].j & 1) ? Xb : Xa) + (long long)job * d_pad * d_pad + (long long)row0 * d_pad;
  double* Rj = R + (long long)job * r_stride;
  const int cols = V2 ? d / 2 : d;
  const long long per = (long long)rows * cols;
  for (long long base = (long long)blockIdx.x * 2048; base < per; base += (long long)gridDim.x * 2048) {
    if (V2) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const long long e = base + u * 256 + threadIdx.x;
        if (e < per) {
          const long long i = e / cols, c = e - i * cols;
          v[u] = *reinterpret_cast<const double2*>(X + i * d_pad + 2 * c);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const long long e = base + u * 256 + threadIdx.x;
        if (e < per) {
          const long long i = e / cols, c = e - i * cols;
          *reinterpret_cast<double2*>(Rj + i * ldr + 2 * c) = v[u];
        }
      }
    } else {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const long long e = base + u * 256 + threadIdx.x;
        if (e < per) {
          const long long i = e / cols, c = e - i * cols;
          v[u] = X[i * d_pad + c];
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const long long e = base + u * 256 + threadIdx.x;
        if (e < per) {
          const long long i = e / cols, c = e - i * cols;
          Rj[i * ldr + c] = v[u];
        }
      }
    }
  }
}

// --------------------------------------------------------------------------------------
// launchers
// --------------------------------------------------------------------------------------
cudaError_t launch_init(const double* H, long long ldh, long long h_stride, double* X, const JobParams* jobs,
                        int d, int d_pad, int batch, cudaStream_t st, int rb0, int rb1) {
  if (rb1 < 0) rb1 = d_pad / 64;
  if (rb1 <= rb0) return cudaSuccess;
  dim3 grid(d_pad / 64, rb1 - rb0, batch);
  ns_init_kernel<<<grid, 256, 0, st>>>(H, ldh, h_stride, X, jobs, d, d_pad, rb0);
  return cudaGetLastError();
}

cudaError_t launch_trace_partials(const double* X, int d, int d_pad, int batch, double* tr_partial,
                                  cudaStream_t st, int job_stride) {
  dim3 grid(d_pad / kTile, batch);
  ns_trace_partials_kernel<<<grid, kTile, 0, st>>>(X, d, d_pad, tr_partial, job_stride);
  return cudaGetLastError();
}

static int diag_tri_env() {
  static const int v = [] {
    const char* e = getenv("NS_DIAG_TRI");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return v;
}

cudaError_t launch_product64(const CUtensorMap& tmP, const CUtensorMap& tmQ, const ProdParams& p_in, int batch,
                             cudaStream_t st) {
  static unsigned long long attr[2] = {0, 0};
  ProdParams p = p_in;
  p.diag_tri = diag_tri_env();
  static const int dbg_sleep = [] { const char* e = getenv("NS_P64_DBG_SLEEP"); return e ? atoi(e) : 0; }();
  static const int dbg_int = [] { const char* e = getenv("NS_P64_DBG_INT"); return e ? atoi(e) : 0; }();
  p.dbg_sleep = dbg_sleep;
  p.dbg_int = dbg_int;
  dim3 grid(p.n_tiles, batch);
  if (p.mode == 0) {
    smem_attr(ns_product64_kernel<0>, k64SmemBytes, attr[0]);
    ns_product64_kernel<0><<<grid, k64Threads, k64SmemBytes, st>>>(tmP, tmQ, p);
  } else {
    smem_attr(ns_product64_kernel<1>, k64SmemBytes, attr[1]);
    ns_product64_kernel<1><<<grid, k64Threads, k64SmemBytes, st>>>(tmP, tmQ, p);
  }
  return cudaGetLastError();
}

cudaError_t launch_product(const CUtensorMap& tmP, const CUtensorMap& tmQ, const ProdParams& p, int batch,
                           cudaStream_t st) {
  static unsigned long long attr[3] = {0, 0, 0};
  dim3 grid(p.n_tiles, batch);
  if (p.mode == 2) {
    smem_attr(ns_product_kernel<2>, kSmemBytes, attr[2]);
    ns_product_kernel<2><<<grid, kThreads, kSmemBytes, st>>>(tmP, tmQ, p);
  } else if (p.mode == 0) {
    smem_attr(ns_product_kernel<0>, kSmemBytes, attr[0]);
    ns_product_kernel<0><<<grid, kThreads, kSmemBytes, st>>>(tmP, tmQ, p);
  } else {
    smem_attr(ns_product_kernel<1>, kSmemBytes, attr[1]);
    ns_product_kernel<1><<<grid, kThreads, kSmemBytes, st>>>(tmP, tmQ, p);
  }
  return cudaGetLastError();
}

cudaError_t launch_decide(DevState* state, const JobParams* jobs, const double* res_partial, int n_tiles,
                          const double* tr_partial, int n_diag, LoopParams lp, int batch, int* n_active,
                          cudaStream_t st, const double* res_ranks, int nranks) {
  ns_decide_kernel<<<batch, 256, 0, st>>>(state, jobs, res_partial, n_tiles, tr_partial, n_diag, lp, n_active,
                                          res_ranks, nranks);
  return cudaGetLastError();
}

cudaError_t launch_copy_out(const double* Xa, const double* Xb, int d, int d_pad, const DevState* state,
                            double* R, long long ldr, long long r_stride, int batch, cudaStream_t st, int row0,
                            int rows) {
  if (rows < 0) rows = d - row0;
  if (rows <= 0) return cudaSuccess;
  const bool v2 = (d % 2 == 0) && (ldr % 2 == 0) && (r_stride % 2 == 0) && ((reinterpret_cast<uintptr_t>(R) & 15) == 0);
  const long long per = (long long)rows * (v2 ? d / 2 : d);
  dim3 grid((unsigned)std::min<long long>((per + 2047) / 2048, 1 << 20), batch);
  if (v2) ns_copy_out_kernel<true><<<grid, 256, 0, st>>>(Xa, Xb, d, d_pad, state, R, ldr, r_stride, row0, rows);
  else ns_copy_out_kernel<false><<<grid, 256, 0, st>>>(Xa, Xb, d, d_pad, state, R, ldr, r_stride, row0, rows);
  return cudaGetLastError();
}

// Stable compaction of the active jobs (batched loop): one CTA, 1024 jobs per pass, warp ballots + a
// scan of the 32 warp counts.  The product kernels then launch only ~n_active CTA rows instead of the
// whole batch (at the tail of configs[1] most rows would otherwise start and exit at once: ~86 us
// per launch for 6144 x 10 empty CTAs).
__global__ void __launch_bounds__(1024) ns_compact_kernel(const DevState* __restrict__ state, int batch,
                                                          int* __restrict__ list, int* __restrict__ n_list) {
  __shared__ int wsum[32];
  __shared__ int carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) carry = 0;
  for (int base = 0; base < batch; base += 1024) {
    __syncthreads();
    const int j = base + tid;
    const bool a = j < batch && !state[j].done;
    const unsigned m = __ballot_sync(0xffffffffu, a);
    if (lane == 0) wsum[warp] = __popc(m);
    __syncthreads();
    if (warp == 0) {
      int v = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      wsum[lane] = v;                       // inclusive
    }
    __syncthreads();
    if (a) list[carry + (warp ? wsum[warp - 1] : 0) + __popc(m & ((1u << lane) - 1u))] = j;
    __syncthreads();
    if (tid == 0) carry += wsum[31];
  }
  __syncthreads();
  if (tid == 0) *n_list = carry;
}

// Speculative result copy (host entry): runs on a side stream next to the square of step jn and
// exits at once unless the decide of step jn - 1 predicted X_jn to be the returned iterate; then it
// streams X_jn to the caller's pinned host R over PCIe, hidden behind that square product.  Few CTAs
// with no shared memory: they fit beside the product kernel's CTA on an SM.
__global__ void __launch_bounds__(256) ns_spec_copy_kernel(const DevState* __restrict__ state, int jn,
                                                           const double* __restrict__ X, int d, int d_pad,
                                                           double* __restrict__ R, long long ldr) {
  if (state->spec != jn) return;
  const int cols = d / 2;   // d even, rows 16-B aligned (checked by the host)
  const long long per = (long long)d * cols;
  for (long long base = (long long)blockIdx.x * 2048; base < per; base += (long long)gridDim.x * 2048) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const long long e = base + u * 256 + threadIdx.x;
      if (e < per) {
        const long long i = e / cols, c = e - i * cols;
        v[u] = *reinterpret_cast<const double2*>(X + i * d_pad + 2 * c);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const long long e = base + u * 256 + threadIdx.x;
      if (e < per) {
        const long long i = e / cols, c = e - i * cols;
        *reinterpret_cast<double2*>(R + i * ldr + 2 * c) = v[u];
      }
    }
  }
}

cudaError_t launch_spec_copy(const DevState* state, int jn, const double* X, int d, int d_pad, double* R,
                             long long ldr, cudaStream_t st) {
  ns_spec_copy_kernel<<<64, 256, 0, st>>>(state, jn, X, d, d_pad, R, ldr);
  return cudaGetLastError();
}

cudaError_t launch_compact(const DevState* state, int batch, int* list, int* n_list, cudaStream_t st) {
  ns_compact_kernel<<<1, 1024, 0, st>>>(state, batch, list, n_list);
  return cudaGetLastError();
}

cudaError_t launch_zero_state(DevState* state, int batch, int* n_active, cudaStream_t st) {
  ns_zero_state_kernel<<<(batch + 255) / 256, 256, 0, st>>>(state, batch, n_active);
  return cudaGetLastError();
}

// Diagnostics (NS_P64_TRACE builds; else returns -1): point the 64-tile kernel's stamps at a device buffer of
// 1 + 10 cap uint64 (buffer[0] must be zeroed by the caller), or turn them off with buf = nullptr.
int p64_trace_set(unsigned long long* buf, unsigned long long cap) {
#if NS_P64_TRACE
  if (cudaMemcpyToSymbol(g_p64_trace, &buf, sizeof(buf)) != cudaSuccess) return -2;
  if (cudaMemcpyToSymbol(g_p64_cap, &cap, sizeof(cap)) != cudaSuccess) return -2;
  return 0;
#else
  (void)buf;
  (void)cap;
  return -1;
#endif
}

}  // namespace nsr
