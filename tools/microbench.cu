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

__global__ void ex2bf2_kernel(float *out, int iters, long long *cyc) {
  uint32_t x[8];
  for (int i = 0; i < 8; ++i) {
    const float a = -(threadIdx.x * 1e-3f + i * 1e-4f), b = a * 0.5f;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(x[i]) : "f"(a), "f"(b));
  }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(x[i]));
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// the softmax pair step with a packed bf16x2 exp: ffma2 -> cvt.bf16x2 (argument) -> ex2.bf16x2 ->
// P ready as bf16x2; row sum: unpack (shift / and) + fadd2
__global__ void pairbf_kernel(float *out, int iters, long long *cyc) {
  uint64_t x[8], acc4[4] = {0, 0, 0, 0}, c2, m2;
  uint32_t pk = 0;
  for (int i = 0; i < 8; ++i) asm("mov.b64 %0, {%1, %1};" : "=l"(x[i]) : "f"(-(threadIdx.x * 1e-3f + i)));
  asm("mov.b64 %0, {%1, %1};" : "=l"(c2) : "f"(0.5f));
  asm("mov.b64 %0, {%1, %1};" : "=l"(m2) : "f"(-0.25f));
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint64_t y;
      asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(y) : "l"(x[i]), "l"(c2), "l"(m2));
      x[i] = y;
      float lo, hi;
      asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(y));
      uint32_t r;
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(r));
      pk ^= r;
      const float p0 = __uint_as_float(r << 16), p1 = __uint_as_float(r & 0xffff0000u);
      asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(p0), "f"(p1));
      asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(acc4[i & 3]) : "l"(y));
    }
  }
  long long t1 = clock64();
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc4[0] ^ acc4[1] ^ acc4[2] ^ acc4[3]));
  out[blockIdx.x * blockDim.x + threadIdx.x] = lo + hi + (float)pk;
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

// cvt.rn.bf16x2.f32 (F2FP.BF16.F32.PACK_AB) throughput
__global__ void f2fp_kernel(float *out, int iters, long long *cyc) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t r;
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x[i]), "f"(x[(i + 1) & 7]));
      x[i] = __uint_as_float(r);
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// the softmax inner step per pair: ffma2, 2 x ex2, fadd2, cvt.bf16x2 (mode 0) or
// the same with the pack done by integer ops (mode 1: add 0x7fff + lsb, prmt)
template <int kMode>
__global__ void pair_kernel(float *out, int iters, long long *cyc) {
  uint64_t x[8], acc4[4] = {0, 0, 0, 0}, c2, m2;
  uint32_t pk = 0;
  for (int i = 0; i < 8; ++i) asm("mov.b64 %0, {%1, %1};" : "=l"(x[i]) : "f"(-(threadIdx.x * 1e-3f + i)));
  asm("mov.b64 %0, {%1, %1};" : "=l"(c2) : "f"(0.5f));
  asm("mov.b64 %0, {%1, %1};" : "=l"(m2) : "f"(-0.25f));
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint64_t y;
      asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(y) : "l"(x[i]), "l"(c2), "l"(m2));
      x[i] = y;
      float lo, hi;
      asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(y));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(lo));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(hi));
      asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(lo), "f"(hi));
      asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(acc4[i & 3]) : "l"(y));
      uint32_t r;
      if (kMode == 0) {
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
      } else {
        const uint32_t a = __float_as_uint(lo) + 0x8000u, b = __float_as_uint(hi) + 0x8000u;
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(a), "r"(b));
      }
      pk ^= r;
    }
  }
  long long t1 = clock64();
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc4[0] ^ acc4[1] ^ acc4[2] ^ acc4[3]));
  out[blockIdx.x * blockDim.x + threadIdx.x] = lo + hi + (float)pk;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename K>
double run(K kern, int warps, int iters, float *out, long long *cyc) {
  long long h[148];
  kern<<<148, warps * 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  return c / 148;
}

int main(int argc, char **argv) {
  if (argc > 1) {  // softmax-step modes only
    float *out; long long *cyc;
    cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
    for (int warps : {4, 8}) {
      const int iters = 2048;
      double c = run(f2fp_kernel, warps, iters, out, cyc);
      printf("cvt.bf16x2 warps/SM=%2d: %.2f cvt/clk/SM\n", warps, warps * 32.0 * iters * 8 / c);
      c = run(pair_kernel<0>, warps, iters, out, cyc);
      printf("pair(cvt)  warps/SM=%2d: %.2f exp/clk/SM  (%.1f cyc per 64-pair row-tile per warp)\n", warps,
             warps * 32.0 * iters * 16 / c, c / iters / 8 * 64 / (warps / 4.0));
      c = run(pairbf_kernel, warps, iters, out, cyc);
      printf("pair(bf16x2 ex2) warps/SM=%2d: %.2f exp/clk/SM  (%.1f cyc per 64-pair row-tile per warp)\n", warps,
             warps * 32.0 * iters * 16 / c, c / iters / 8 * 64 / (warps / 4.0));
      c = run(pair_kernel<1>, warps, iters, out, cyc);
      printf("pair(prmt) warps/SM=%2d: %.2f exp/clk/SM  (%.1f cyc per 64-pair row-tile per warp)\n", warps,
             warps * 32.0 * iters * 16 / c, c / iters / 8 * 64 / (warps / 4.0));
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
  }
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
    ex2bf2_kernel<<<148, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
    c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
    printf("ex2 bf16x2 warps/SM=%2d: %.2f exp/clk/SM (2 per op)\n", warps, (double)warps * 32 * iters * 8 * 2 / c);
    ffma2_kernel<<<148, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
    c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
    printf("ffma2 warps/SM=%2d: %.2f fp32-fma/clk/SM (packed x2)\n", warps, (double)warps * 32 * iters * 8 * 2 / c);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
