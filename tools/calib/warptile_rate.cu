// Calibration: DMMA.8x8x4 throughput of the K loop alone, fragments read from shared memory in the tiled
// kernels' layout (128-byte swizzle, k-permuted LDS.128: one load gives a lane two k-steps), for different
// warp tiles and warps per SM.  No TMA, no epilogue, no ring barriers: the question is what the inner loop
// shape itself sustains (the 64x64-tile kernel uses 32x32 warp tiles and reaches ~83-87% DMMA activity at
// configs[1], the 128x128-tile kernel 64x32 warp tiles and 98.6% at d = 16384).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 warptile_rate.cu -o warptile_rate
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

__device__ __forceinline__ void lds128(uint32_t addr, double& x, double& y) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(addr));
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
      : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// MI x NI fragments of 8x8 per warp; operands: a slab of 128 rows x 16 doubles for A and for B (32 KB)
template <int MI, int NI>
__global__ void loop_kernel(int iters, double* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  double* s = reinterpret_cast<double*>(smem);
  for (int i = threadIdx.x; i < 2 * 128 * 16; i += blockDim.x) s[i] = 1e-3 * (i % 13);
  __syncthreads();
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const uint32_t off0 = ((2 * t) ^ g) << 4, off1 = ((2 * t + 1) ^ g) << 4;
  const uint32_t a_row = base + ((warp * 8 * MI) % 128 + g) * 128;
  const uint32_t b_row = base + 128 * 16 * 8 + ((warp * 8 * NI) % 128 + g) * 128;
  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t off = h ? off1 : off0;
      double a[MI][2], b[NI][2];
#pragma unroll
      for (int j = 0; j < NI; ++j) lds128(b_row + j * 8 * 128 + off, b[j][0], b[j][1]);
#pragma unroll
      for (int i = 0; i < MI; ++i) lds128(a_row + i * 8 * 128 + off, a[i][0], a[i][1]);
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NI; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i][e], b[j][e]);
    }
  }
  double sum = 0.0;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) sum += acc[i][j][0] + acc[i][j][1];
  if (sum == 12345.0) out[threadIdx.x] = sum;
}

template <int MI, int NI>
void run(const char* name, int warps, int ctas_per_sm, double* out) {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int smem = 2 * 128 * 16 * 8 + 1024;
  cudaFuncSetAttribute(loop_kernel<MI, NI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4000, blocks = sms * ctas_per_sm;
  loop_kernel<MI, NI><<<blocks, 32 * warps, smem>>>(10, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  loop_kernel<MI, NI><<<blocks, 32 * warps, smem>>>(iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flop = 2.0 * 256.0 * 4.0 * MI * NI * (double)iters * blocks * warps;   // 4 k-steps per iteration
  const double tf = flop / (ms * 1e-3) / 1e12;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, loop_kernel<MI, NI>, 32 * warps, smem);
  printf("%-34s warps/CTA %d  CTAs/SM %d (occ %d)  %7.2f TFLOP/s  %5.1f%% of 36.97\n", name, warps, ctas_per_sm, occ, tf,
         100.0 * tf / 36.97);
  (void)clk;
}

int main() {
  double* out;
  cudaMalloc(&out, 4096 * sizeof(double));
  run<4, 4>("32x32 warp tile (64-tile kernel)", 4, 3, out);
  run<4, 4>("32x32 warp tile", 4, 4, out);
  run<4, 4>("32x32 warp tile", 8, 2, out);
  run<8, 4>("64x32 warp tile (128-tile kernel)", 8, 1, out);
  run<8, 4>("64x32 warp tile", 4, 2, out);
  run<8, 4>("64x32 warp tile", 2, 4, out);
  run<8, 4>("64x32 warp tile", 2, 6, out);
  run<4, 2>("32x16 warp tile", 8, 3, out);
  run<2, 4>("16x32 warp tile", 4, 3, out);
  // one and two K-loop warps per SM sub-partition (what a CTA sustains while its co-residents are outside their K loops)
  run<4, 4>("32x32 warp tile, 1 warp/SMSP", 4, 1, out);
  run<4, 4>("32x32 warp tile, 2 warps/SMSP", 4, 2, out);
  run<8, 4>("64x32 warp tile, 1 warp/SMSP", 4, 1, out);
  run<4, 8>("32x64 warp tile, 1 warp/SMSP", 4, 1, out);
  run<4, 8>("32x64 warp tile, 2 warps/SMSP", 4, 2, out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
  return 0;
}
