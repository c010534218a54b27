// gather_bench.cu — per-SM throughput of the three ways to stream 128-row x 256-B
// (bf16 d = 128) key tiles into shared memory through a row permutation:
//   mode 0: TMA tile load of contiguous rows (the permuted-copy path)
//   mode 1: TMA tile::gather4 through the permutation (4 rows / instruction)
//   mode 2: cp.async 16 B per lane through the permutation (LDGSTS), mbarrier completion
// One CTA per SM, one producer warp, a 4-stage ring; a consumer warp only waits
// and releases.  Reports GB/s per SM and aggregate.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t *b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void mexpect(uint64_t *b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void marrive(uint64_t *b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory"); }
__device__ __forceinline__ void mwait(uint64_t *b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su(b)), "r"(ph) : "memory");
}

constexpr int ROWS = 128, STAGES = 4;
constexpr uint32_t TILE = ROWS * 256;

template <int kMode>
__global__ void __launch_bounds__(64, 1) bench(const __grid_constant__ CUtensorMap tile_map, const __grid_constant__ CUtensorMap g_map,
                                               const char *src, const int *perm, int n_rows, int tiles, long long *cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { minit(&full[s], kMode == 2 ? 32 : 1); minit(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t base = su(sm);
  long long t0 = clock64();
  if (warp == 0) {
    for (int t = 0; t < tiles; ++t) {
      const int s = t % STAGES;
      mwait(&empty[s], ((t / STAGES) & 1) ^ 1);
      const int row0 = (int)((((long long)blockIdx.x * 7919 + t * 131) * ROWS) % (n_rows - ROWS));
      if (kMode == 0) {
        if (lane == 0) {
          mexpect(&full[s], TILE);
          for (int bx = 0; bx < 2; ++bx)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(base + s * TILE + bx * (TILE / 2)), "l"((uint64_t)&tile_map), "r"(bx * 64), "r"(row0), "r"(su(&full[s])) : "memory");
        }
      } else if (kMode == 1) {
        int r[4];
        for (int i = 0; i < 4; ++i) r[i] = __ldg(perm + row0 + 4 * lane + i);
        if (lane == 0) mexpect(&full[s], TILE);
        __syncwarp();
        for (int bx = 0; bx < 2; ++bx)
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                       ::"r"(base + s * TILE + bx * (TILE / 2) + lane * 512), "l"((uint64_t)&g_map), "r"(bx * 64), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(su(&full[s])) : "memory");
      } else {
        // 128 rows x 16 chunks of 16 B: lane handles chunk (lane & 15) of rows (lane >> 4) + 2i
        for (int i = 0; i < ROWS / 2; ++i) {
          const int row = (lane >> 4) + 2 * i, ch = lane & 15;
          const int pr = __ldg(perm + row0 + row);
          const char *g = src + (size_t)pr * 256 + ch * 16;
          const int bx = ch >> 3, c8 = ch & 7;
          const uint32_t dst = base + s * TILE + bx * (TILE / 2) + row * 128 + ((c8 ^ (row & 7)) << 4);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(g) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su(&full[s])) : "memory");
      }
    }
  } else if (lane == 0) {
    for (int t = 0; t < tiles; ++t) {
      const int s = t % STAGES;
      mwait(&full[s], (t / STAGES) & 1);
      marrive(&empty[s]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  const int n_rows = 32 * 32768;  // 32 heads x 32K tokens, 256 B per row (1 GB... 256 MB)
  char *src; int *perm; long long *cyc;
  cudaMalloc(&src, (size_t)n_rows * 256);
  cudaMemset(src, 1, (size_t)n_rows * 256);
  std::vector<int> hp(n_rows);
  for (int i = 0; i < n_rows; ++i) hp[i] = i;
  srand(1);
  for (int h = 0; h < 32; ++h)  // permute within each head (like pi_k)
    for (int i = 32767; i > 0; --i) { int j = rand() % (i + 1); std::swap(hp[h * 32768 + i], hp[h * 32768 + j]); }
  cudaMalloc(&perm, n_rows * 4);
  cudaMemcpy(perm, hp.data(), n_rows * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&cyc, 148 * 8);
  void *fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap tm, gm;
  cuuint64_t dims[2] = {128, (cuuint64_t)n_rows}, str[1] = {256};
  cuuint32_t box[2] = {64, ROWS}, gbox[2] = {64, 1}, es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&gm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, str, gbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int tiles = 400;
  const size_t smem = STAGES * TILE;
  auto run = [&](auto kern, const char *name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 2; ++rep) {
      kern<<<148, 64, smem>>>(tm, gm, src, perm, n_rows, tiles, cyc);
      cudaDeviceSynchronize();
    }
    long long h[148];
    cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
    double c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
    printf("%-28s %7.1f cycles/tile  %6.1f B/clk/SM  (%s)\n", name, c / tiles, TILE * (double)tiles / c, cudaGetErrorString(cudaGetLastError()));
  };
  run(bench<0>, "TMA tile (contiguous)");
  run(bench<1>, "TMA gather4 (through pi)");
  run(bench<2>, "cp.async 16B (through pi)");
  return 0;
}
