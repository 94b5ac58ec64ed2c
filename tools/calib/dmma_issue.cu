// Calibration: does a non-DMMA instruction cost DMMA throughput?  Each warp runs DMMA.8x8x4 from registers
// (16 independent accumulators) with E extra instructions per DMMA of a chosen kind interleaved in the same
// warp (integer ALU, FP32, shared-memory loads, FP64 FMA), at 1, 2 and 3 warps per SM sub-partition.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 dmma_issue.cu -o dmma_issue
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// KIND 0: none, 1: integer (LOP3/IADD chain x E), 2: LDS.128 x E, 3: DFMA x E, 4: FFMA x E
template <int KIND, int E>
__global__ void k(int iters, double* out) {
  __shared__ double sm[1024];
  sm[threadIdx.x & 1023] = threadIdx.x;
  __syncthreads();
  double acc[16][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = 1e-3 * threadIdx.x, b = 2e-3;
  unsigned x0 = threadIdx.x, x1 = 7, x2 = 9, x3 = 11;
  float f0 = 1.f, f1 = 2.f, f2 = 3.f, f3 = 4.f;
  double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
  double l0 = 0.0, l1 = 0.0;
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(sm)) + (threadIdx.x & 31) * 16;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      dmma(acc[i][0], acc[i][1], a, b);
#pragma unroll
      for (int q = 0; q < E; ++q) {
        if (KIND == 1) {
          if ((q & 3) == 0) asm volatile("lop3.b32 %0, %0, %1, 0x5a5a5a5a, 0x96;" : "+r"(x0) : "r"(x1));
          if ((q & 3) == 1) asm volatile("add.u32 %0, %0, %1;" : "+r"(x1) : "r"(x2));
          if ((q & 3) == 2) asm volatile("lop3.b32 %0, %0, %1, 0x33333333, 0x96;" : "+r"(x2) : "r"(x3));
          if ((q & 3) == 3) asm volatile("add.u32 %0, %0, %1;" : "+r"(x3) : "r"(x0));
        } else if (KIND == 2) {
          double u, v;
          asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(u), "=d"(v) : "r"(sbase + ((i * E + q) & 7) * 512));
          l0 += 0;  // keep registers
          if (q == 0) { l0 = u; l1 = v; }
        } else if (KIND == 3) {
          if ((q & 3) == 0) asm volatile("fma.rn.f64 %0, %1, %1, %0;" : "+d"(e0) : "d"(a));
          if ((q & 3) == 1) asm volatile("fma.rn.f64 %0, %1, %1, %0;" : "+d"(e1) : "d"(b));
          if ((q & 3) == 2) asm volatile("fma.rn.f64 %0, %1, %1, %0;" : "+d"(e2) : "d"(a));
          if ((q & 3) == 3) asm volatile("fma.rn.f64 %0, %1, %1, %0;" : "+d"(e3) : "d"(b));
        } else if (KIND == 4) {
          if ((q & 3) == 0) asm volatile("fma.rn.f32 %0, %1, %1, %0;" : "+f"(f0) : "f"(f1));
          if ((q & 3) == 1) asm volatile("fma.rn.f32 %0, %1, %1, %0;" : "+f"(f1) : "f"(f2));
          if ((q & 3) == 2) asm volatile("fma.rn.f32 %0, %1, %1, %0;" : "+f"(f2) : "f"(f3));
          if ((q & 3) == 3) asm volatile("fma.rn.f32 %0, %1, %1, %0;" : "+f"(f3) : "f"(f0));
        }
      }
    }
  }
  double sum = e0 + e1 + e2 + e3 + l0 + l1 + (double)(x0 + x1 + x2 + x3) + (double)(f0 + f1 + f2 + f3);
#pragma unroll
  for (int i = 0; i < 16; ++i) sum += acc[i][0] + acc[i][1];
  if (sum == 12345.678) out[threadIdx.x] = sum;
}

template <int KIND, int E>
void run(const char* name, int warps_per_smsp, double* out) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4000, threads = 128 * warps_per_smsp;
  k<KIND, E><<<sms, threads>>>(10, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<KIND, E><<<sms, threads>>>(iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  const double flop = 2.0 * 256.0 * 16.0 * iters * (threads / 32.0) * sms;
  const double tf = flop / (ms * 1e-3) / 1e12;
  printf("%-22s E=%2d  warps/SMSP %d  %7.2f TFLOP/s  %5.1f%% of 36.97\n", name, E, warps_per_smsp, tf, 100.0 * tf / 36.97);
}

int main() {
  double* out;
  cudaMalloc(&out, 8192 * sizeof(double));
  for (int w = 1; w <= 3; ++w) {
    run<0, 0>("DMMA only", w, out);
    run<1, 1>("+ integer", w, out);
    run<1, 2>("+ integer", w, out);
    run<1, 4>("+ integer", w, out);
    run<1, 8>("+ integer", w, out);
    run<1, 16>("+ integer", w, out);
    run<2, 1>("+ LDS.128", w, out);
    run<2, 2>("+ LDS.128", w, out);
    run<3, 1>("+ DFMA", w, out);
    run<3, 2>("+ DFMA", w, out);
    run<3, 4>("+ DFMA", w, out);
    run<4, 4>("+ FFMA", w, out);
    run<4, 8>("+ FFMA", w, out);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
  return 0;
}
