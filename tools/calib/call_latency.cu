// Calibration: host wall time per ns_reflector call on a d=64 problem straight through the C ABI (no
// Python), to split call latency into library/driver overhead and kernel time.
// build: nvcc -O2 -std=c++17 -I../../include call_latency.cu -o call_latency -L../../paper_2605_24840_b200
//        -lnsreflector -Xlinker -rpath=$PWD/../../paper_2605_24840_b200
#include <chrono>
#include <cmath>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

#include "nsreflector.h"

__global__ void empty_kernel(int* flag) {
  if (flag && threadIdx.x == 0) {
    __threadfence_system();
    *(volatile int*)flag = 1;
  }
}

int main() {
  const int d = 64;
  std::vector<double> h(d * d, 0.0);
  for (int i = 0; i < d; ++i) h[i * d + i] = (i < 3) ? -1.0 : 1.0;   // diagonal: 3 negative eigenvalues
  for (int i = 0; i + 1 < d; ++i) h[i * d + i + 1] = h[(i + 1) * d + i] = 0.01;
  double *H, *R;
  void* ws;
  cudaMalloc(&H, d * d * 8);
  cudaMalloc(&R, d * d * 8);
  const size_t wsb = ns_workspace_bytes(d, NS_PREC_FP64);
  cudaMalloc(&ws, wsb);
  cudaMemcpy(H, h.data(), d * d * 8, cudaMemcpyHostToDevice);
  ns_result_t res;
  for (int m : {0, 8}) {
    for (int i = 0; i < 20; ++i) ns_reflector(H, d, d, 0.0, 1.2, 3, m, 0.0, NS_TOL_ABS, NS_PREC_FP64, R, d, ws, wsb, nullptr, &res);
    const int n = 2000;
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) ns_reflector(H, d, d, 0.0, 1.2, 3, m, 0.0, NS_TOL_ABS, NS_PREC_FP64, R, d, ws, wsb, nullptr, &res);
    auto t1 = std::chrono::steady_clock::now();
    printf("C ABI ns_reflector d=64 max_steps=%d: %.1f us per call (steps %d cert %lld)\n", m,
           std::chrono::duration<double, std::micro>(t1 - t0).count() / n, res.steps, (long long)res.index_cert);
  }
  // bare launch + sync latency of an empty kernel, and launch + host spin on a flag the kernel writes to mapped
  // pinned memory, for reference
  {
    const int n = 2000;
    for (int i = 0; i < 20; ++i) empty_kernel<<<1, 32>>>(nullptr);
    cudaDeviceSynchronize();
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) {
      empty_kernel<<<1, 32>>>(nullptr);
      cudaStreamSynchronize(nullptr);
    }
    auto t1 = std::chrono::steady_clock::now();
    printf("empty kernel launch + cudaStreamSynchronize: %.1f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / n);
    volatile int* hflag;
    int* dflag;
    cudaHostAlloc((void**)&hflag, 4, cudaHostAllocMapped);
    cudaHostGetDevicePointer((void**)&dflag, (void*)hflag, 0);
    t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) {
      *hflag = 0;
      empty_kernel<<<1, 32>>>(dflag);
      while (*hflag == 0) {
      }
    }
    t1 = std::chrono::steady_clock::now();
    cudaDeviceSynchronize();
    printf("empty kernel launch + host spin on a mapped flag: %.1f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / n);
  }
  return 0;
}
