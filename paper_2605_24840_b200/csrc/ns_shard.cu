// Multi-GPU Newton–Schulz for large d (BASELINE configs[4]):
// one process per GPU.
//
// Partitioning: every rank keeps the full iterate X (replicated, 8 d_pad^2 bytes) but computes only
// its share of the n(n+1)/2 upper 128x128 output tiles of each symmetric product:
// rank r owns tiles t of the L2-ordered upper-tile list with t % P == r (balanced to one tile).
//
// Default exchange (ns_api.cu run_sharded + ns_fp64.cu epilogue): every rank's workspace is mapped
// into every process through CUDA IPC, and the product kernel's epilogue stores each tile, its mirror
// and its residual / trace partial into all ranks' buffers over NVLink as the tile finishes; a
// one-double ncclAllReduce per product is the barrier.  This file holds the kernels of the fallback
// exchange (NCCL all-gather, used when a rank cannot map its peers):
//   1. Y tiles (own) <- X X               ns_product_kernel<0> on the rank's tile list
//   2. residual partials -> one double    ns_shard_sum_kernel (fixed order)
//   3. the rank's tile list is cut into C chunks; as soon as chunk c's product kernel finishes (event
//      on the compute stream) a communication stream packs its tiles, all-gathers them (NCCL) and
//      unpacks the other ranks' copies into Y (mirrored) while chunk c+1 is being computed, so the
//      exchange overlaps the contraction chunk by chunk; + ncclAllGather of the P residual sums
//      (summed in rank order: identical bits on all ranks)
//   4. the compute stream waits for the last unpack before anything reads the full Y
//   5. decide (identical on all ranks)
//   6. X_{j+1} tiles (own) <- 1.5 X - 0.5 X Y, pack, all-gather, unpack; tr X_{j+1} locally.
// Communication per step: 2 all-gathers of d^2/2 doubles (each rank receives (P-1)/P of them)
// + 2 x P doubles; compute per rank 2 d^3 / P.  At d = 49152, P = 8: ~19 GB/step received vs
// ~0.85 s of DMMA work per step (~3% on NVLink 5 before overlap).
#include <cstdint>

#include "ns_internal.h"
#include "ns_ptx.cuh"

namespace nsr {

// Copy the rank's tiles (local list entries 0..n_my-1) of the d_pad x d_pad matrix M into the
// tile-major send buffer (tile t -> send[t * 128*128 ...], row-major inside the tile).
__global__ void __launch_bounds__(256) ns_pack_tiles_kernel(const double* __restrict__ M, const int2* __restrict__ my_tiles,
                                                            double* __restrict__ send, int d_pad) {
  const int2 tl = my_tiles[blockIdx.x];
  const double* src = M + (long long)tl.x * kTile * d_pad + (long long)tl.y * kTile;
  double* dst = send + (long long)blockIdx.x * kTile * kTile;
  for (int i = threadIdx.x; i < kTile * kTile / 2; i += 256) {
    const int r = (2 * i) >> 7, c = (2 * i) & 127;
    const double2 v = *reinterpret_cast<const double2*>(src + (long long)r * d_pad + c);
    *reinterpret_cast<double2*>(dst + (long long)r * kTile + c) = v;
  }
}

// Scatter every other rank's gathered tiles of one chunk into M, with the mirrored block for
// off-diagonal tiles.  grid = (cs, P): slot s of rank q in chunk c holds the rank's local tile
// slot0 + s, i.e. global upper tile (slot0 + s) * P + q (absent if >= n_tiles).
__global__ void __launch_bounds__(256) ns_unpack_tiles_kernel(double* __restrict__ M, const int2* __restrict__ all_tiles,
                                                              int n_tiles, const double* __restrict__ recv_chunk,
                                                              int cs, int slot0, int nranks, int my_rank, int d_pad) {
  __shared__ double t[32][33];
  const int q = blockIdx.y, slot = blockIdx.x;
  if (q == my_rank) return;
  const long long gt = (long long)(slot0 + slot) * nranks + q;
  if (gt >= n_tiles) return;
  const int2 tl = all_tiles[gt];
  const double* src = recv_chunk + ((long long)q * cs + slot) * kTile * kTile;
  double* dst = M + (long long)tl.x * kTile * d_pad + (long long)tl.y * kTile;
  for (int i = threadIdx.x; i < kTile * kTile / 2; i += 256) {
    const int r = (2 * i) >> 7, c = (2 * i) & 127;
    *reinterpret_cast<double2*>(dst + (long long)r * d_pad + c) = *reinterpret_cast<const double2*>(src + r * kTile + c);
  }
  if (tl.x == tl.y) return;
  // mirror: M[J*128 + c][I*128 + r] = tile[r][c], through 32x32 smem transposes
  double* mdst = M + (long long)tl.y * kTile * d_pad + (long long)tl.x * kTile;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int bi = 0; bi < 4; ++bi)
    for (int bj = 0; bj < 4; ++bj) {
      __syncthreads();
      for (int y = ty; y < 32; y += 8) t[y][tx] = src[(bi * 32 + y) * kTile + bj * 32 + tx];
      __syncthreads();
      for (int y = ty; y < 32; y += 8) mdst[(long long)(bj * 32 + y) * d_pad + bi * 32 + tx] = t[tx][y];
    }
}

// out[0] = sum_{i < n} v[i] in a fixed order (one block).
__global__ void __launch_bounds__(256) ns_shard_sum_kernel(const double* __restrict__ v, int n, double* out) {
  __shared__ double red[8];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) s += v[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    out[0] = t;
  }
}

// Receiver-side mirror: the peer-store epilogue (remote_mirror = 0) sends only the upper tile (I, J) to the
// other ranks; after the barrier each rank fills M[J-block][I-block] = M[I-block][J-block]^T for the tiles it
// did not compute itself (its own tiles were mirrored by its own epilogue).  One CTA per tile of the global
// list, 32x32 shared-memory transposes (coalesced reads and writes).
__global__ void __launch_bounds__(256) ns_mirror_remote_kernel(double* __restrict__ M, const int2* __restrict__ all_tiles,
                                                               int nranks, int my_rank, int d_pad) {
  __shared__ double t[32][33];
  const int gt = blockIdx.x;
  if (gt % nranks == my_rank) return;
  const int2 tl = all_tiles[gt];
  if (tl.x == tl.y) return;
  const double* src = M + (long long)tl.x * kTile * d_pad + (long long)tl.y * kTile;
  double* dst = M + (long long)tl.y * kTile * d_pad + (long long)tl.x * kTile;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int bi = 0; bi < 4; ++bi)
    for (int bj = 0; bj < 4; ++bj) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = src[(long long)(bi * 32 + ty + 8 * u) * d_pad + bj * 32 + tx];
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 4; ++u) t[ty + 8 * u][tx] = v[u];
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 4; ++u) dst[(long long)(bj * 32 + ty + 8 * u) * d_pad + bi * 32 + tx] = t[tx][ty + 8 * u];
    }
}

// Block-row initial iterate (ns_reflector_sharded_rows): rank r holds rows [r0, r1) of H.  Block (bj, by)
// covers the 64x64 tile (bi, bj), bi = r0/64 + by, of the global matrix; only tiles with bj >= bi and only
// elements (i, j) with r0 <= i < r1, i <= j < d are read (the upper triangle of the rank's rows).  Each
// element x = (H_ij - s delta_ij)/alpha is stored at (i, j) and (j, i) in every destination (every rank's
// X_0 through the peer mappings), so after the barrier all ranks hold the full symmetric X_0.
__global__ void __launch_bounds__(256) ns_init_rows_kernel(const double* __restrict__ Hr, long long ldh, long long r0,
                                                           long long r1, double* const* __restrict__ dst, int n_dst,
                                                           double s, double alpha, int d, int d_pad) {
  __shared__ double t[64][65];
  const int bj = blockIdx.x;
  const int bi = (int)(r0 / 64) + blockIdx.y;
  if (bj < bi) return;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;   // 64 x 4
  double v[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const long long gi = (long long)bi * 64 + ty + 4 * u, gj = (long long)bj * 64 + tx;
    double x = 0.0;
    if (gi >= r0 && gi < r1 && gj >= gi && gj < d) {
      const double h = Hr[(gi - r0) * ldh + gj];
      x = (gi == gj) ? (h - s) / alpha : h / alpha;
    }
    v[u] = x;
    t[ty + 4 * u][tx] = x;
  }
  __syncthreads();
  for (int q = 0; q < n_dst; ++q) {
    double* X = dst[q];
#pragma unroll
    for (int u = 0; u < 16; ++u) {   // direct: (i, j), j >= i
      const long long gi = (long long)bi * 64 + ty + 4 * u, gj = (long long)bj * 64 + tx;
      if (gi >= r0 && gi < r1 && gj >= gi && gj < d) X[gi * d_pad + gj] = v[u];
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {   // mirror: row j = bj*64 + ty + 4u, column i = bi*64 + tx, for j > i
      const long long gj = (long long)bj * 64 + ty + 4 * u, gi = (long long)bi * 64 + tx;
      if (gi >= r0 && gi < r1 && gj > gi && gj < d) X[gj * d_pad + gi] = t[tx][ty + 4 * u];
    }
  }
}

cudaError_t launch_mirror_remote(double* M, const int2* all_tiles, int n_tiles, int nranks, int my_rank, int d_pad,
                                 cudaStream_t st) {
  if (nranks > 1 && n_tiles > 0) ns_mirror_remote_kernel<<<n_tiles, 256, 0, st>>>(M, all_tiles, nranks, my_rank, d_pad);
  return cudaGetLastError();
}

cudaError_t launch_init_rows(const double* H_rows, long long ldh, long long r0, long long r1, double* const* dst,
                             int n_dst, double s, double alpha, int d, int d_pad, cudaStream_t st) {
  if (r1 <= r0) return cudaSuccess;
  const int rb0 = (int)(r0 / 64), rb1 = (int)((r1 + 63) / 64);
  dim3 grid(d_pad / 64, rb1 - rb0);
  ns_init_rows_kernel<<<grid, 256, 0, st>>>(H_rows, ldh, r0, r1, dst, n_dst, s, alpha, d, d_pad);
  return cudaGetLastError();
}

cudaError_t launch_pack_tiles(const double* M, const int2* my_tiles, int n_my, double* send, int d_pad,
                              cudaStream_t st) {
  if (n_my > 0) ns_pack_tiles_kernel<<<n_my, 256, 0, st>>>(M, my_tiles, send, d_pad);
  return cudaGetLastError();
}

cudaError_t launch_unpack_tiles(double* M, const int2* all_tiles, int n_tiles, const double* recv_chunk, int cs,
                                int slot0, int nranks, int my_rank, int d_pad, cudaStream_t st) {
  if (nranks > 1 && cs > 0) {
    dim3 grid(cs, nranks);
    ns_unpack_tiles_kernel<<<grid, 256, 0, st>>>(M, all_tiles, n_tiles, recv_chunk, cs, slot0, nranks, my_rank, d_pad);
  }
  return cudaGetLastError();
}

cudaError_t launch_shard_sum(const double* v, int n, double* out, cudaStream_t st) {
  ns_shard_sum_kernel<<<1, 256, 0, st>>>(v, n, out);
  return cudaGetLastError();
}

}  // namespace nsr
