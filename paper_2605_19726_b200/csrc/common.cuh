// common.cuh — small device helpers shared by the BA-Att kernels (sm_100a).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define BA_DEVICE __device__ __forceinline__

namespace baatt {

constexpr int kWarp = 32;

// Convert a 16-byte chunk into EPC floats (EPC = 16 / sizeof(T)).
template <typename T> struct Chunk;
template <> struct Chunk<float> {
  static constexpr int EPC = 4;
  BA_DEVICE static void unpack(const uint4 &u, float (&f)[4]) {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
  }
};
template <> struct Chunk<__nv_bfloat16> {
  static constexpr int EPC = 8;
  BA_DEVICE static void unpack(const uint4 &u, float (&f)[8]) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);            // low half = element 2i
      f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);  // high half = element 2i+1
    }
  }
};

BA_DEVICE int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
BA_DEVICE int imax(int a, int b) { return a > b ? a : b; }

BA_DEVICE uint4 ldg16(const void *p) { return __ldg(reinterpret_cast<const uint4 *>(p)); }
BA_DEVICE void stg16(void *p, const uint4 &v) { *reinterpret_cast<uint4 *>(p) = v; }

BA_DEVICE float to_float(float x) { return x; }
BA_DEVICE float to_float(__nv_bfloat16 x) { return __bfloat162float(x); }

// Order-preserving map of an fp64 value onto uint64 (ascending).
BA_DEVICE uint64_t ordered_bits(double x) {
  uint64_t u = static_cast<uint64_t>(__double_as_longlong(x));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

BA_DEVICE unsigned lanemask_lt() {
  unsigned m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace baatt
