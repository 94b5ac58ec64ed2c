// Calibration: device time of one fused small-d product (ns_small.cu small_ns_product) on one SM,
// repeated back to back, to separate the contraction from the per-step scalar work.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2605_24840_b200/csrc
//        small_prod_bench.cu -o small_prod_bench
#include <cstdio>

#include "../../paper_2605_24840_b200/csrc/ns_small.cu"

using namespace nsr;

template <int DP, int MODE, bool SYNC>
__global__ void __launch_bounds__(small_threads<DP>(), 1) bench(int reps, double* out) {
  constexpr int P = small_pitch<DP>();
  extern __shared__ __align__(16) double sm[];
  double* X = sm;
  double* Y = sm + DP * P;
  double* C = sm + 2 * DP * P;
  __shared__ int2 units[small_units<DP>()];
  small_fill_units<DP>(units);
  for (int e = threadIdx.x; e < DP * P; e += blockDim.x) {
    X[e] = 1e-3 * (e % 7);
    Y[e] = 1e-3 * (e % 5);
  }
  __syncthreads();
  double acc = 0.0;
  for (int r = 0; r < reps; ++r) {
    acc += small_ns_product<DP, MODE>(X, Y, C, DP, 1.5, -0.5, units);
    if (SYNC) __syncthreads();
  }
  out[threadIdx.x] = acc + C[threadIdx.x];
}

template <int DP, int MODE, bool SYNC>
void run(const char* name) {
  const size_t smem = 3 * DP * small_pitch<DP>() * sizeof(double);
  cudaFuncSetAttribute(bench<DP, MODE, SYNC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  double* out;
  cudaMalloc(&out, 4096 * sizeof(double));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  bench<DP, MODE, SYNC><<<1, small_threads<DP>(), smem>>>(10, out);
  const int reps = 2000;
  cudaEventRecord(a);
  bench<DP, MODE, SYNC><<<1, small_threads<DP>(), smem>>>(reps, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double frags = (DP / 8) * (DP / 8 + 1) / 2.0;
  const double flop = frags * 64.0 * DP * 2.0;
  printf("%-28s DP=%3d threads=%4d  %.3f us/product  %.1f%% of one SM's FP64 peak (%.0f GF/s/SM)\n", name, DP,
         small_threads<DP>(), 1e3 * ms / reps, 100.0 * flop / (ms * 1e-3 / reps) / (37.2e12 / 148),
         flop / (ms * 1e-3 / reps) / 1e9);
  cudaFree(out);
}

int main() {
  run<32, 0, true>("square+sync");
  run<64, 0, true>("square+sync");
  run<64, 0, false>("square nosync");
  run<64, 1, true>("update+sync");
  run<96, 0, true>("square+sync");
  run<96, 1, true>("update+sync");
  return 0;
}
