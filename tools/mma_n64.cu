// mma_n64.cu — tcgen05 rate of the S MMA at N = 64 vs N = 128 (M = 128, K = 16,
// SS form, bf16 -> fp32): is a 64-key S sub-tile issued at the full tensor rate?
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
#include "../paper_2605_19726_b200/csrc/sm100_ptx.cuh"
using namespace baatt::sm100;

template <int N>
__global__ void __launch_bounds__(128, 1) s_kernel(int iters, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t ID = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
  if (threadIdx.x == 0) {
    const uint32_t sq = base, sk = base + 32768;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int h = 0; h < 128 / N; ++h) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          mma_ss(tmem + (it & 1) * 128 + h * N, make_desc(sq + off, 16, 1024),
                 make_desc(sk + off + h * N * 128, 16, 1024), ID, kk > 0);
        }
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

int main() {
  long long *d, h[148];
  cudaMalloc(&d, 148 * 8);
  const int iters = 4000, smem = 70 * 1024;
  cudaFuncSetAttribute(s_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(s_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) {
    s_kernel<128><<<148, 128, smem>>>(iters, d);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("S N=128: %.1f cycles per 128x128x128 S (floor 512)\n", (double)h[0] / iters);
    s_kernel<64><<<148, 128, smem>>>(iters, d);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("S N=64 x2: %.1f cycles per 128x128x128 S (floor 512)\n", (double)h[0] / iters);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
