// attn_simt.cu — K6: block-sparse attention on CUDA cores (fp32 math).
//
// The fp32 path of Alg. 1 steps 11-12: for every query row i of
// query block g_q, softmax over the keys of the selected blocks only,
// O'_i = sum_j P_ij V'_j, streamed with an online softmax, then written to the
// original row pi_q(i).  Used for fp32 inputs (config T, 1e-5 parity)
// and as the correct-but-slow path for bf16 shapes the tensor-core kernel does
// not cover.  One CTA per (batch*head, g_q); one thread per query row; K/V
// staged through shared memory 32 keys at a time.
#include <math.h>

#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace baatt {

constexpr int kSimtThreads = 128;  // >= block size B
constexpr int kSimtChunk = 32;     // keys per smem stage

template <typename T, int D>
__global__ void __launch_bounds__(kSimtThreads) attn_simt_kernel(AttnArgs a) {
  // fp32 inputs accumulate O and l in fp64: fp32 accumulation over ~1e3 keys
  // costs ~3e-5 absolute, above the 1e-5 gate of the fp32 config.
  using Acc = typename std::conditional<sizeof(T) == 4, double, float>::type;
  extern __shared__ __align__(16) float sm[];
  float *Qs = sm;                                  // [128][D+1]
  float *Ks = Qs + kSimtThreads * (D + 1);         // [32][D+1]
  float *Vs = Ks + kSimtChunk * (D + 1);           // [32][D]
  const int64_t gq = blockIdx.x;
  const int64_t bh = blockIdx.y;
  const int64_t b = bh / a.hq, h = bh - b * a.hq;
  const int64_t grp = a.hq / a.hkv;
  const int64_t hk = h / grp;
  const int i = threadIdx.x;
  const int64_t row0 = gq * a.B;
  const int nqrows = (int)imin64(a.B, a.lq - row0);
  const T *q = static_cast<const T *>(a.q) + b * a.qs[0] + h * a.qs[1];
  const T *k = static_cast<const T *>(a.k) + b * a.ks[0] + hk * a.ks[1];
  const T *v = static_cast<const T *>(a.v) + b * a.vs[0] + hk * a.vs[1];
  for (int e = threadIdx.x; e < nqrows * D; e += kSimtThreads) {
    const int r = e / D, c = e - r * D;
    Qs[r * (D + 1) + c] = to_float(q[(row0 + r) * a.qs[2] + c]);
  }
  const int64_t row = (bh * a.nq + gq);
  const int cnt = a.kv_index ? (a.kv_count ? a.kv_count[row] : (int)a.kv_stride) : (int)a.nk;
  if (cnt < 1 && threadIdx.x == 0) flag_error(a.err_flag, kErrEmptyRow);  // S:393; rows -> O = 0, LSE = -inf
  double m = -INFINITY;
  Acc l = 0;
  Acc acc[D];
#pragma unroll
  for (int c = 0; c < D; ++c) acc[c] = 0;
  for (int s = 0; s < cnt; ++s) {
    const int64_t gk = a.kv_index ? a.kv_index[row * a.kv_stride + s] : s;
    if (gk < 0 || gk >= a.nk) {  // uniform across the CTA: every thread reads the same entry
      if (threadIdx.x == 0) flag_error(a.err_flag, kErrBadIndex);
      continue;
    }
    const int64_t k0 = gk * a.B;
    const int nk = (int)imin64(a.B, a.lk - k0);
    for (int c0 = 0; c0 < nk; c0 += kSimtChunk) {
      const int n = min(kSimtChunk, nk - c0);
      __syncthreads();
      for (int e = threadIdx.x; e < n * D; e += kSimtThreads) {
        const int r = e / D, c = e - r * D;
        const int64_t tok = k0 + c0 + r;
        Ks[r * (D + 1) + c] = to_float(k[tok * a.ks[2] + c]);
        Vs[r * D + c] = to_float(v[tok * a.vs[2] + c]);
      }
      __syncthreads();
      if (i < nqrows) {
        // logits in fp64 (exact products of fp32 values): large fp32 logits would
        // otherwise cost ~1e-7 * |logit| absolute, too much for the 1e-5 gate
        double sc[kSimtChunk];
        double cmax = -INFINITY;
#pragma unroll
        for (int jj = 0; jj < kSimtChunk; ++jj) {
          double dot = 0.0;
          if (jj < n) {
#pragma unroll 16
            for (int c = 0; c < D; ++c) dot = fma((double)Qs[i * (D + 1) + c], (double)Ks[jj * (D + 1) + c], dot);
            dot *= (double)a.scale;
            cmax = fmax(cmax, dot);
          }
          sc[jj] = dot;
        }
        const double mn = fmax(m, cmax);
        const Acc corr = (Acc)exp(m - mn);  // m = -inf on the first chunk -> 0
        l *= corr;
#pragma unroll
        for (int c = 0; c < D; ++c) acc[c] *= corr;
#pragma unroll
        for (int jj = 0; jj < kSimtChunk; ++jj) {
          if (jj < n) {
            const Acc p = sizeof(Acc) == 8 ? (Acc)exp(sc[jj] - mn) : (Acc)expf((float)(sc[jj] - mn));
            l += p;
#pragma unroll 16
            for (int c = 0; c < D; ++c) acc[c] = fma(p, (Acc)Vs[jj * D + c], acc[c]);
          }
        }
        m = mn;
      }
    }
  }
  if (i < nqrows) {
    const int64_t srow = row0 + i;
    const int64_t orow = a.perm_q ? a.perm_q[bh * a.lq + srow] : srow;
    T *o = static_cast<T *>(a.out) + b * a.os[0] + h * a.os[1] + orow * a.os[2];
    const Acc inv = l > (Acc)0 ? (Acc)1 / l : (Acc)0;  // empty row: O = 0, LSE = -inf
#pragma unroll
    for (int c = 0; c < D; ++c) {
      if constexpr (sizeof(T) == 4) o[c] = (float)(acc[c] * inv);
      else o[c] = __float2bfloat16_rn((float)(acc[c] * inv));
    }
    if (a.lse) a.lse[bh * a.lq + orow] = l > (Acc)0 ? (float)(m + log((double)l)) : -INFINITY;
  }
}

cudaError_t launch_attn_simt(const AttnArgs &a, cudaStream_t st) {
  dim3 grid((unsigned)a.nq, (unsigned)(a.batch * a.hq));
#define BA_SIMT(T, D)                                                                                 \
  do {                                                                                                \
    const size_t smem = sizeof(float) * (kSimtThreads * (D + 1) + kSimtChunk * (D + 1) + kSimtChunk * D); \
    cudaError_t e = cudaFuncSetAttribute(attn_simt_kernel<T, D>,                                      \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);    \
    if (e != cudaSuccess) return e;                                                                   \
    attn_simt_kernel<T, D><<<grid, kSimtThreads, smem, st>>>(a);                                      \
  } while (0)
  if (a.dtype == 1 && a.d == 64) BA_SIMT(float, 64);
  else if (a.dtype == 1 && a.d == 128) BA_SIMT(float, 128);
  else if (a.dtype == 0 && a.d == 64) BA_SIMT(__nv_bfloat16, 64);
  else BA_SIMT(__nv_bfloat16, 128);
#undef BA_SIMT
  return cudaGetLastError();
}

}  // namespace baatt
