// FP64 pipe calibration on sm_100a: DMMA (mma.sync .f64 shapes) and DFMA
// throughput per SM, measured with CUDA events over a full-chip grid.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_calib fp64_calib.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int NACC>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dmma_m16n8k4(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-9, a1 = a0 * 0.5, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_k(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <typename K>
static int run(const char* name, K kern, int blocks, int threads, int iters, double fma_per_thread_iter,
               double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, 10);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double fmas = fma_per_thread_iter * (double)blocks * threads * iters;
  int dev; cudaGetDevice(&dev);
  int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double tflops = 2.0 * fmas / (best * 1e-3) / 1e12;
  printf("%-28s blocks=%4d thr=%4d  %8.3f ms  %7.2f TFLOP/s  %6.1f FMA/clk/SM @%d MHz (attr)\n", name, blocks,
         threads, best, tflops, fmas / (best * 1e-3) / sms / (clk_khz * 1e3), clk_khz / 1000);
  return 0;
}

int main() {
  double* out;
  CK(cudaMalloc(&out, 1 << 20));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s  SMs %d  cc %d.%d\n", p.name, sms, p.major, p.minor);
  const int it = 4000;
  // m8n8k4: 256 FMA per warp-instr -> 8 FMA per thread per mma
  for (int w : {4, 8, 16}) {
    run("dmma m8n8k4 x8acc", dmma_m8n8k4<8>, sms, 32 * w, it, 8.0 * 8, out);
  }
  run("dmma m8n8k4 x4acc", dmma_m8n8k4<4>, sms, 32 * 8, it, 8.0 * 4, out);
  run("dmma m8n8k4 x16acc", dmma_m8n8k4<16>, sms, 32 * 8, it / 2, 8.0 * 16, out);
  run("dmma m8n8k4 x8acc 2blk/SM", dmma_m8n8k4<8>, sms * 2, 32 * 8, it, 8.0 * 8, out);
  // m16n8k4: 512 FMA per warp-instr -> 16 FMA per thread
  for (int w : {4, 8}) run("dmma m16n8k4 x8acc", dmma_m16n8k4<8>, sms, 32 * w, it, 16.0 * 8, out);
  for (int w : {4, 8, 16}) run("dfma x8", dfma_k<8>, sms, 32 * w, it * 4, 8.0, out);
  run("dfma x16 1024thr", dfma_k<16>, sms, 1024, it * 2, 16.0, out);
  return 0;
}
