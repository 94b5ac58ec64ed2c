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
// CTA = 6 warps: warp 0 TMA producer, warp 1 MMA issuer (one elected lane; owns the TMEM
// allocation), warps 2..5 epilogue (warp w reads TMEM lane quadrant w % 4).  128x128 output tile,
// UMMA M=128 N=128 K=16, 6-stage ring of 32 KB (A and B: 128 rows x 64 bf16, 128-B swizzle).
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

__global__ void __launch_bounds__(256) ns_split_planes_kernel(const double* __restrict__ X,
                                                              uint16_t* __restrict__ planes, long long n_per_job,
                                                              int batch) {
  const long long total = n_per_job * batch;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long job = i / n_per_job, e = i - job * n_per_job;
    uint16_t hi, lo;
    split_bf16(X[i], hi, lo);
    planes[job * 2 * n_per_job + e] = hi;
    planes[job * 2 * n_per_job + n_per_job + e] = lo;
  }
}

template <int MODE>
__global__ void __launch_bounds__(kMxThreads, 1)
    ns_mx_product_kernel(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmQ,
                         const MxParams p) {
  const int job = blockIdx.y;
  if (p.state != nullptr && p.state[job].done) return;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                        // [stages][128 x 64 bf16]
  uint8_t* sB = smem + kMxStages * kTile * kMxBK * 2;        // [stages][128 x 64 bf16]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kMxStages * kMxStageBytes);
  uint64_t* empty = full + kMxStages;
  uint64_t* tmem_full = empty + kMxStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  __shared__ double red[4];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int2 tile = p.tiles[blockIdx.x];
  const int I = tile.x, J = tile.y;
  const int nkb_total = 3 * p.nkb;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 128);
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
        const int seg = kb / p.nkb, kk = kb - seg * p.nkb;
        const int pa = (seg == 1) ? 1 : 0;   // segments: (hi,lo), (lo,hi), (hi,hi)
        const int pb = (seg == 0) ? 1 : 0;
        mbar_arrive_expect_tx(&full[s], kMxStageBytes);
        tma_load_3d(sA + s * kTile * kMxBK * 2, &tmP, kk * kMxBK, I * kTile, 2 * job + pa, &full[s]);
        tma_load_3d(sB + s * kTile * kMxBK * 2, &tmQ, kk * kMxBK, J * kTile, 2 * job + pb, &full[s]);
      }
    }
  } else if (warp == 1) {
    // idesc: D=F32 (bits 4-5 = 1), A=B=BF16 (bits 7-9, 10-12 = 1), K-major, N=128 (>>3 at 17), M=128 (>>4 at 24)
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kTile >> 3) << 17) |
                           ((uint32_t)(kTile >> 4) << 24);
    for (int kb = 0; kb < nkb_total; ++kb) {
      const int s = kb % kMxStages;
      mbar_wait(&full[s], static_cast<uint32_t>(kb / kMxStages) & 1u);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t a0 = smem_u32(sA + s * kTile * kMxBK * 2);
        const uint32_t b0 = smem_u32(sB + s * kTile * kMxBK * 2);
#pragma unroll
        for (int k = 0; k < kMxBK / 16; ++k)
          umma_bf16(tmem, sdesc_k128(a0 + k * 32), sdesc_k128(b0 + k * 32), idesc, (kb | k) != 0);
        umma_commit(&empty[s]);
        if (kb == nkb_total - 1) umma_commit(tmem_full);
      }
      __syncwarp();
    }
  } else {
    // ---------------- epilogue: TMEM -> FP64 -> smem staging -> global ----------------
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const int q = warp & 3;                 // TMEM lane quadrant of this warp
    const int r = q * 32 + lane;            // tile row owned by this thread
    double* S = reinterpret_cast<double*>(smem);   // [128][kEpiPitch]; the ring is idle once tmem_full fired
#pragma unroll 1
    for (int c0 = 0; c0 < kTile; c0 += 32) {
      uint32_t v[32];
      tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) S[r * kEpiPitch + c0 + i] = (double)__uint_as_float(v[i]);
    }
  }
  // all roles: ring no longer in use (epilogue wrote S only after the last MMA completed)
  tc_fence_before();
  __syncthreads();

  if (warp >= 2) {
    double* S = reinterpret_cast<double*>(smem);
    const int tid = threadIdx.x - 64;       // 0..127
    const long long ld = p.ld;
    const long long base = (long long)job * p.job_stride;
    double* C = p.C + base;
    const long long nplane = (long long)p.ld * p.ld;
    uint16_t* Ph = p.Cplanes ? p.Cplanes + (long long)job * 2 * nplane : nullptr;
    uint16_t* Pl = Ph ? Ph + nplane : nullptr;
    const bool diag = (I == J);
    double part = 0.0;
    auto put = [&](long long gidx, double v) {
      C[gidx] = v;
      if (Ph) {
        uint16_t h, l;
        split_bf16(v, h, l);
        Ph[gidx] = h;
        Pl[gidx] = l;
      }
    };
    if (MODE == 2) {
      for (int idx = tid; idx < kTile * kTile; idx += 128) {
        const int rr = idx >> 7, cc = idx & 127;
        put((long long)(I * kTile + rr) * ld + J * kTile + cc, S[rr * kEpiPitch + cc]);
      }
    } else if (MODE == 0) {
      if (!diag) {
        for (int idx = tid; idx < kTile * kTile; idx += 128) {
          const int rr = idx >> 7, cc = idx & 127;
          const double v = S[rr * kEpiPitch + cc];
          put((long long)(I * kTile + rr) * ld + J * kTile + cc, v);
          part += v * v;
        }
        part *= 2.0;
        for (int idx = tid; idx < kTile * kTile; idx += 128) {
          const int rr = idx >> 7, cc = idx & 127;
          put((long long)(J * kTile + rr) * ld + I * kTile + cc, S[cc * kEpiPitch + rr]);
        }
      } else {
        for (int idx = tid; idx < kTile * kTile; idx += 128) {
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
        for (int idx = tid; idx < kTile * kTile; idx += 128) {
          const int rr = idx >> 7, cc = idx & 127;
          const long long g = (long long)(I * kTile + rr) * ld + J * kTile + cc;
          const double v = fma(-0.5, S[rr * kEpiPitch + cc], 1.5 * X[g]);
          put(g, v);
          S[rr * kEpiPitch + cc] = v;
        }
        named_bar_sync(1, 128);
        for (int idx = tid; idx < kTile * kTile; idx += 128) {
          const int rr = idx >> 7, cc = idx & 127;
          put((long long)(J * kTile + rr) * ld + I * kTile + cc, S[cc * kEpiPitch + rr]);
        }
      } else {
        for (int idx = tid; idx < kTile * kTile; idx += 128) {
          const int rr = idx >> 7, cc = idx & 127;
          if (rr <= cc) {
            const long long g = (long long)(I * kTile + rr) * ld + I * kTile + cc;
            const double v = fma(-0.5, S[rr * kEpiPitch + cc], 1.5 * X[g]);
            S[rr * kEpiPitch + cc] = v;
            if (rr == cc && I * kTile + rr < p.d) part += v;
          }
        }
        named_bar_sync(1, 128);
        for (int idx = tid; idx < kTile * kTile; idx += 128) {
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
      named_bar_sync(1, 128);
      if (tid == 0) {
        const double s = ((red[0] + red[1]) + red[2]) + red[3];
        if (MODE == 0) p.partial[(long long)job * p.n_tiles + blockIdx.x] = s;
        else if (diag) p.partial[(long long)job * (p.ld / kTile) + I] = s;
      }
    }
  }
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 128);
}

cudaError_t launch_split_planes(const double* X, uint16_t* planes, int d_pad, int batch, cudaStream_t st) {
  const long long n = (long long)d_pad * d_pad;
  long long blocks = (n * batch + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  ns_split_planes_kernel<<<(unsigned)blocks, 256, 0, st>>>(X, planes, n, batch);
  return cudaGetLastError();
}

cudaError_t launch_mx_product(const CUtensorMap& tmP, const CUtensorMap& tmQ, const MxParams& p, int batch,
                              cudaStream_t st) {
  static bool attr[3] = {false, false, false};
  dim3 grid(p.n_tiles, batch);
  switch (p.mode) {
    case 0:
      if (!attr[0]) { cudaFuncSetAttribute(ns_mx_product_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMxSmemBytes); attr[0] = true; }
      ns_mx_product_kernel<0><<<grid, kMxThreads, kMxSmemBytes, st>>>(tmP, tmQ, p);
      break;
    case 1:
      if (!attr[1]) { cudaFuncSetAttribute(ns_mx_product_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMxSmemBytes); attr[1] = true; }
      ns_mx_product_kernel<1><<<grid, kMxThreads, kMxSmemBytes, st>>>(tmP, tmQ, p);
      break;
    default:
      if (!attr[2]) { cudaFuncSetAttribute(ns_mx_product_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMxSmemBytes); attr[2] = true; }
      ns_mx_product_kernel<2><<<grid, kMxThreads, kMxSmemBytes, st>>>(tmP, tmQ, p);
      break;
  }
  return cudaGetLastError();
}

}  // namespace nsr
