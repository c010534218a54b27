// mma_bench.cu — tcgen05 issue/execute rate for the attention kernel's MMA mix,
// operands resident (no TMA, no softmax): cycles per (S = Q K^T, O += P V) pair.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
#include "../paper_2605_19726_b200/csrc/sm100_ptx.cuh"
using namespace baatt::sm100;

// 0: S TS + PV TS, 1: S SS + PV TS, 2: S SS only, 3: PV TS only,
// 4: mode 0 + a commit after each 8-MMA group, 5: mode 4 + fence + wait on a completed barrier per group
// 11: mode 8 without the tcgen05 fence after the K-full wait, 12: mode 8 without any tcgen05 fence after waits
// 6: the kernel's handoff: S_{j+1} issued, then wait for warp 1 to see S_j complete and arrive, then PV_j
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
  uint32_t r;
  asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
               : "=r"(r) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return r != 0;
}

// 15: mode 9 without the MMA thread's K-full wait (producer and commits unchanged; data race irrelevant here)
// 17: mode 7 + one extra commit (kempty) after PV; 18: mode 16 with the two commits issued before PV instead of after
// 16: mode 7 + the kempty / odone commits of mode 9 (no producer, no K-full wait)
// 14: mode 9 with the producer polling its empty barrier by test_wait + nanosleep(128) instead of try_wait
// 13: mode 9 with a CUTLASS-style peek: the K-full barrier of S(j+2) is tested (non-blocking) in the middle of
//     PV(j)'s MMAs and the blocking wait before S(j+2) is skipped when it was already complete
template <int MODE>
__global__ void __launch_bounds__(352, 1) mma_kernel(int iters, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t raw = smem_u32(sm), base = (raw + 1023u) & ~1023u;
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t cbar[4];
  __shared__ __align__(8) uint64_t sfull[2], pfull[2];
  __shared__ __align__(8) uint64_t kfull[4], kempty[4], vfull[2], vempty[2], odone;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&cbar[i], 1);
    mbar_init(&cbar[3], 1);
    for (int i = 0; i < 2; ++i) { mbar_init(&sfull[i], 1); mbar_init(&pfull[i], MODE >= 7 ? 8 : 1); }
    for (int i = 0; i < 4; ++i) { mbar_init(&kfull[i], 1); mbar_init(&kempty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&vfull[i], 1); mbar_init(&vempty[i], 1); }
    mbar_init(&odone, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t IDS = (1u << 4) | (1u << 7) | (1u << 10) | (16u << 17) | (8u << 24);
  const uint32_t IDO = IDS | (1u << 16);
  long long t0 = 0, t1 = 0;
  constexpr bool P8 = MODE == 8 || MODE == 11 || MODE == 12;  // modes 11-12 are mode 8 variants
  constexpr bool P9 = MODE == 9 || MODE == 10 || MODE == 13 || MODE == 14 || MODE == 15;
  bool peeked = false;
  if (MODE >= 6) {
    if (threadIdx.x == 0) {
      const uint32_t sk = base + 32768, sv = base + 65536;
      auto issue_s = [&](int j) {
        if (MODE >= 8 && MODE != 15 && MODE < 16 && !(MODE == 10 && j >= 2) && !(MODE == 13 && peeked)) { mbar_wait(&kfull[j & 3], (j >> 2) & 1); if (MODE < 11) tc_fence_after(); }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          mma_ts(tmem + (j & 1) * 128, tmem + 384 + kk * 8, make_desc(sk + off, 16, 1024), IDS, kk > 0);
        }
        if (P8) mma_commit(&kempty[j & 3]);
        mma_commit(&sfull[j & 1]);
      };
      t0 = clock64();
      issue_s(0);
      for (int j = 0; j < iters; ++j) {
        if (j + 1 < iters) issue_s(j + 1);
        mbar_wait(&pfull[j & 1], (j >> 1) & 1);
        if (P8) mbar_wait(&vfull[j & 1], (j >> 1) & 1);  // MODE 9: V arrived with K (kfull)
        if (MODE != 12) tc_fence_after();
        if (MODE == 18) { mma_commit(&kempty[j & 3]); mma_commit(&odone); }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (MODE == 10 && kk == 4 && j + 2 < iters) { mbar_wait(&kfull[(j + 2) & 3], ((j + 2) >> 2) & 1); tc_fence_after(); }
          if (MODE == 13 && kk == 4) peeked = j + 2 < iters && mbar_test(&kfull[(j + 2) & 3], ((j + 2) >> 2) & 1);
          mma_ts(tmem + 256, tmem + (j & 1) * 128 + kk * 8, make_desc(sv + kk * 2048, 16384, 1024), IDO, 1);
        }
        if (P8) { mma_commit(&vempty[j & 1]); mma_commit(&odone); }
        if (P9 || MODE == 16) { mma_commit(&kempty[j & 3]); mma_commit(&odone); }
        if (MODE == 17) mma_commit(&kempty[j & 3]);
      }
      mma_commit(&bar);
      mbar_wait(&bar, 0);
      t1 = clock64();
      out[blockIdx.x] = t1 - t0;
    } else if (P9 && threadIdx.x == 320) {
      for (int j = 0; j < iters; ++j) {
        if (MODE == 14) { while (!mbar_test(&kempty[j & 3], ((j >> 2) & 1) ^ 1)) __nanosleep(128); }
        else mbar_wait(&kempty[j & 3], ((j >> 2) & 1) ^ 1);
        mbar_arrive(&kfull[j & 3]);
      }
    } else if (P8 && (threadIdx.x == 320 || threadIdx.x == 32)) {
      // producers without data: wait for the free slot, arrive on the full barrier (K: 4 stages, V: 2)
      const bool is_k = threadIdx.x == 320;
      for (int j = 0; j < iters; ++j) {
        if (is_k) { mbar_wait(&kempty[j & 3], ((j >> 2) & 1) ^ 1); mbar_arrive(&kfull[j & 3]); }
        else { mbar_wait(&vempty[j & 1], ((j >> 1) & 1) ^ 1); mbar_arrive(&vfull[j & 1]); }
      }
    } else if ((MODE == 6 && threadIdx.x == 32) || (MODE >= 7 && threadIdx.x >= 64 && threadIdx.x < 320)) {
      // MODE 7: 8 warps (256 threads) wait like the softmax warpgroups, one elected arrive per warp
      for (int j = 0; j < iters; ++j) {
        mbar_wait(&sfull[j & 1], (j >> 1) & 1);
        tc_fence_after();
        tc_fence_before();
        if (MODE >= 7) __syncwarp();
        if (MODE == 6 || (threadIdx.x & 31) == 0) mbar_arrive(&pfull[j & 1]);
      }
    }
  } else if (threadIdx.x == 0) {
    const uint32_t sq = base, sk = base + 32768, sv = base + 65536;
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t sc = (it % 3) * 128;
      if (MODE != 3) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          if (MODE == 0 || MODE >= 4) mma_ts(tmem + sc, tmem + 384 + kk * 8, make_desc(sk + off, 16, 1024), IDS, kk > 0);
          else mma_ss(tmem + sc, make_desc(sq + off, 16, 1024), make_desc(sk + off, 16, 1024), IDS, kk > 0);
        }
      }
      if (MODE != 2) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(tmem + 384 - 128 * (MODE == 0 || MODE >= 4), tmem + sc + kk * 8, make_desc(sv + kk * 2048, 16384, 1024), IDO, 1);
      }
      if (MODE >= 4) { mma_commit(&cbar[0]); mma_commit(&cbar[1]); }
      if (MODE == 5) { mbar_wait(&cbar[3], 1); tc_fence_after(); }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

int main() {
  long long *d, h[148];
  cudaMalloc(&d, 148 * 8);
  const int iters = 2000;
  const char *names[4] = {"S TS + PV TS", "S SS + PV TS", "S SS only   ", "PV TS only  "};
  const char *names2[19] = {"S TS + PV TS", "S SS + PV TS", "S SS only   ", "PV TS only  ", "+commits    ", "+commit+wait", "handoff     ", "handoff x8w ", "+producers  ", "+1 kv ring  ", "kv wait mid ", "8 - kfence  ", "8 - fences  ", "9 + peek    ", "9 + sleepy p", "9 - kwait   ", "7 + commits ", "7 + 1 commit", "7 + 2c early"};
  for (int mode = 0; mode < 19; ++mode) {
    auto k = mode == 0 ? mma_kernel<0> : mode == 1 ? mma_kernel<1> : mode == 2 ? mma_kernel<2> : mode == 3 ? mma_kernel<3> : mode == 4 ? mma_kernel<4> : mode == 5 ? mma_kernel<5> : mode == 6 ? mma_kernel<6> : mode == 7 ? mma_kernel<7> : mode == 8 ? mma_kernel<8> : mode == 9 ? mma_kernel<9> : mode == 10 ? mma_kernel<10> : mode == 11 ? mma_kernel<11> : mode == 12 ? mma_kernel<12> : mode == 13 ? mma_kernel<13> : mode == 14 ? mma_kernel<14> : mode == 15 ? mma_kernel<15> : mode == 16 ? mma_kernel<16> : mode == 17 ? mma_kernel<17> : mma_kernel<18>;

    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int rep = 0; rep < 2; ++rep) {
      k<<<148, 352, 100 * 1024>>>(iters, d);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
    double c = 0;
    for (int i = 0; i < 148; ++i) c += h[i];
    c /= 148;
    const int mmas = (mode < 2 || mode >= 4 ? 16 : 8);  // mode 6: S + PV per iteration
    printf("%s: %.1f cycles per iteration (%d MMAs of 128x128x16) = %.1f cyc/MMA (floor 64)\n", names2[mode], c / iters, mmas, c / iters / mmas);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
