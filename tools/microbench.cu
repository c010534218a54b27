// microbench.cu — measures B200 unit throughputs that bound the attention kernel:
// MUFU.EX2 per SM per clock, FFMA2 per SM per clock.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void ex2_kernel(float *out, int iters, long long *cyc) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void ex2h2_kernel(float *out, int iters, long long *cyc) {
  uint32_t x[8];
  for (int i = 0; i < 8; ++i) {
    const float a = -(threadIdx.x * 1e-3f + i * 1e-4f), b = a * 0.5f;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(x[i]) : "f"(a), "f"(b));
  }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x[i]));
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void ffma2_kernel(float *out, int iters, long long *cyc) {
  uint64_t x[8];
  for (int i = 0; i < 8; ++i) asm("mov.b64 %0, {%1, %1};" : "=l"(x[i]) : "f"(threadIdx.x * 1e-3f + i));
  uint64_t a, c;
  asm("mov.b64 %0, {%1, %1};" : "=l"(a) : "f"(0.999f));
  asm("mov.b64 %0, {%1, %1};" : "=l"(c) : "f"(0.001f));
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(a), "l"(c));
  }
  long long t1 = clock64();
  float s = 0, lo, hi;
  for (int i = 0; i < 8; ++i) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[i])); s += lo + hi; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float *out; long long *cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  long long h[148];
  for (int warps : {1, 2, 4, 8, 16}) {
    const int iters = 4096;
    ex2_kernel<<<148, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
    double c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
    printf("ex2   warps/SM=%2d: %.2f ex2/clk/SM\n", warps, (double)warps * 32 * iters * 8 / c);
    ex2h2_kernel<<<148, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
    c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
    printf("ex2 f16x2 warps/SM=%2d: %.2f exp/clk/SM (2 per op)\n", warps, (double)warps * 32 * iters * 8 * 2 / c);
    ffma2_kernel<<<148, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
    c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
    printf("ffma2 warps/SM=%2d: %.2f fp32-fma/clk/SM (packed x2)\n", warps, (double)warps * 32 * iters * 8 * 2 / c);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
