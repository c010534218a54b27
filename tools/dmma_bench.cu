// dmma_bench.cu — FP64 throughput on B200: DFMA (SIMT) vs mma.sync.m8n8k4.f64 (DMMA).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double *out, int iters, long long *cyc) {
  double x[8], a = 1.0000001, c = 1e-9;
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, c);
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void dmma_kernel(double *out, int iters, long long *cyc) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.5, c[4][2];
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  double *out; long long *cyc, h[148];
  cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&cyc, 148 * 8);
  for (int warps : {4, 8, 16, 32}) {
    const int iters = 2048;
    dfma_kernel<<<148, warps * 32>>>(out, iters, cyc); cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
    double c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
    printf("dfma warps/SM=%2d: %6.1f FLOP/clk/SM\n", warps, warps * 32.0 * iters * 8 * 2 / c);
    dmma_kernel<<<148, warps * 32>>>(out, iters, cyc); cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
    c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
    printf("dmma warps/SM=%2d: %6.1f FLOP/clk/SM\n", warps, warps * iters * 4 * 512.0 / c);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
