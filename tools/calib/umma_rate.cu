// Calibration: issue rate of tcgen05.mma kind::f16 (BF16, FP32 accumulate) and kind::i8 for M=128 and
// N = 64 / 128 / 256 (cta_group::1), operands resident in shared memory, back to back into TMEM.
// Reports MACs per SM clock (dense BF16 nominal: 2.25 PF / 148 SMs / 1.965 GHz / 2 = 3868 MAC/clk).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 umma_rate.cu -o umma_rate
#include <cstdio>
#include <cstdint>

#include "../../paper_2605_24840_b200/csrc/ns_ptx.cuh"

using namespace nsr;

__device__ __forceinline__ uint64_t sdesc128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

template <int N, bool I8>
__global__ void __launch_bounds__(128, 1) bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if ((threadIdx.x >> 5) == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t a = smem_u32(smem), b = a + 128 * 128;
  // kind::f16: D=F32 (1<<4), A=B=BF16 (1<<7, 1<<10); kind::i8: D=S32 (2<<4), signed
  const uint32_t idesc = (I8 ? ((2u << 4) | (1u << 7) | (1u << 10)) : ((1u << 4) | (1u << 7) | (1u << 10))) |
                         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t ad = sdesc128(a + k * 32), bd = sdesc128(b + k * 32);
        if (I8)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(ad), "l"(bd),
                       "r"(idesc), "r"(1u) : "memory");
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(ad), "l"(bd),
                       "r"(idesc), "r"(1u) : "memory");
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) tmem_dealloc(tmem, 512);
}

template <int N, bool I8>
void run() {
  const int iters = 4096, smem = (128 + 256) * 128 + 2048;
  cudaFuncSetAttribute(bench<N, I8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  bench<N, I8><<<148, 128, smem>>>(16, d);
  bench<N, I8><<<148, 128, smem>>>(iters, d);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double k_per = I8 ? 32.0 : 16.0;   // K per instruction
  const double macs = (double)iters * 4 * 128.0 * N * k_per;
  printf("%s M=128 N=%3d K=%2.0f: %7.1f cycles per UMMA, %7.0f MAC/clk/SM\n", I8 ? "i8 " : "f16", N, k_per,
         mx / (iters * 4.0), macs / mx);
  cudaFree(d);
}

int main() {
  run<64, false>();
  run<128, false>();
  run<256, false>();
  run<64, true>();
  run<128, true>();
  run<256, true>();
  return 0;
}
