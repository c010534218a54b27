// block_mass_sm100.cu — NEXT-3 fidelity diagnostic on the tensor cores: the
// oracle block distribution (Eq. oracle-dist)
//
//   m_hat[g_q, g_k] = (1/|I(g_q)|) sum_{i in I(g_q)} sum_{j in J(g_k)} A_ij,
//   A = softmax(Q' K'^T * scale)  (dense, over every key of the row),
//
// in the norm-sorted block space the selection ranks, and the
// captured mass of the selection, sum_{g_k : M = 1} m_hat[g_q, g_k] (the
// quantity the paper's Fig. 2 / ablation compare m' against).
//
// The row normaliser comes from a dense pass of the attention kernel over
// the same Q', K', V' (its LSE output), so A_ij = 2^(s_ij * c - lse2_i) with
// c = scale * log2(e) and lse2 = lse * log2(e).  This kernel recomputes
// S = Q' K'^T tile by tile on tcgen05 (no PV MMA) and reduces exp over the
// 128 x 128 tile in registers, warp shuffles and 8 partials in smem.
//
// The same S pass also yields, per block pair, the extremes of the token
// logits S_ij = Q'_i . K'_j over the block pair's valid rows and columns: the
// "observed maximum logit deviation" max |l_hat_ij - l| of Fig. 2 (P:386-392,
// Eq. logit-deviation) is max(S_max/sqrt(d) - l, l - S_min/sqrt(d)).
// Template flags: kMass (the exp reduction; needs the LSE) and kExt (extremes).
//
// One CTA per 128-row query block (B = 128, bf16, d = 128).  10 warps:
//   warp 0  TMA producer of the K tiles of EVERY key block (4-stage ring);
//   warp 1  TMEM owner, MMA issuer (S_j = Q K_j^T, Q held in TMEM as the A
//           operand, double-buffered S), and the reducer: after the 8 mass
//           warps' partials of tile j land it writes m_hat and accumulates
//           the captured mass over the selected blocks (smem bitmask);
//   warps 2-9  two warpgroups splitting the 128 columns of each row.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "sm100_ptx.cuh"

namespace baatt {
namespace sm100 {

bool make_map(CUtensorMap *m, const void *ptr, int64_t b, int64_t H, int64_t L, int64_t d, const int64_t *s, int rows);
PFN_cuTensorMapEncodeTiled_v12000 get_encode();

namespace mass {

constexpr int BM = 128, BN = 128, HD = 128;
constexpr uint32_t BOX = 128 * 64 * 2, TILE = 2 * BOX;  // 128 rows x 128 bf16 (two 64-column boxes)
constexpr int NST = 4;                                   // K ring stages
constexpr uint32_t Q_COL = 384;                          // TMEM: S0 [0,128), S1 [128,256), Q [384,448)
constexpr int kThreads = 320;
constexpr int kMaskWords = 1024;                         // selection bitmask: N_k <= 32768
constexpr uint32_t SMEM_K = 0;
constexpr uint32_t SMEM_PART = SMEM_K + NST * TILE;       // float [3][2][8] tile partials (mass, max, min)
constexpr uint32_t SMEM_MASK = SMEM_PART + 3 * 2 * 8 * 4; // uint32 [kMaskWords]
constexpr uint32_t SMEM_BARS = SMEM_MASK + kMaskWords * 4;
constexpr uint32_t SMEM_BYTES = SMEM_BARS + 256 + 1024;   // + alignment slack
// kind::f16, D fp32, A/B bf16, K-major both, M = 128, N = 128
constexpr uint32_t IDESC_S = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

struct __align__(8) Bars {
  uint64_t q_full;
  uint64_t full[NST], empty[NST];
  uint64_t s_full[2], p_full[2];
  uint32_t tmem_base;
};

template <bool kMass, bool kExt>
__global__ void __launch_bounds__(kThreads, 1)
block_mass_kernel(const MassArgs a, const __grid_constant__ CUtensorMap tm_k) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t *smem = smem_raw + (base - raw);
  Bars &bars = *reinterpret_cast<Bars *>(smem + SMEM_BARS);
  float *part = reinterpret_cast<float *>(smem + SMEM_PART);
  uint32_t *sel = reinterpret_cast<uint32_t *>(smem + SMEM_MASK);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gq = blockIdx.x, bh = blockIdx.y;
  const int64_t b = bh / a.hq, h = bh - b * a.hq;
  const int64_t hk = h / (a.hq / a.hkv);
  const int cnt = (int)a.nk;  // dense: every key block
  const int64_t row0 = gq * BM;
  const int nrows = (int)imin64(BM, a.lq - row0);

  for (int w = threadIdx.x; w < kMaskWords; w += kThreads) sel[w] = 0u;
  __syncthreads();
  if (a.kv_index) {  // the selection whose captured mass is reported
    const int64_t row = bh * a.nq + gq;
    const int c = a.kv_count ? a.kv_count[row] : (int)a.kv_stride;
    for (int e = threadIdx.x; e < c; e += kThreads) {
      const int g = a.kv_index[row * a.kv_stride + e];
      if ((unsigned)g < (unsigned)a.nk) atomicOr(&sel[g >> 5], 1u << (g & 31));  // out-of-range entries ignored
    }
  }
  if (threadIdx.x == 0) {
    mbar_init(&bars.q_full, 8);
    for (int s = 0; s < NST; ++s) { mbar_init(&bars.full[s], 1); mbar_init(&bars.empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&bars.s_full[s], 1); mbar_init(&bars.p_full[s], 8); }
    fence_barrier_init();
    tma_prefetch(&tm_k);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&bars.tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;

  if (warp == 0) {
    // ================================================================ TMA producer (K only)
    if (lane == 0) {
      for (int j = 0; j < cnt; ++j) {
        const int s = j % NST;
        mbar_wait(&bars.empty[s], ((uint32_t)(j / NST) & 1u) ^ 1u);
        const uint32_t dk = base + SMEM_K + s * TILE;
        mbar_expect_tx(&bars.full[s], TILE);
        tma_load_4d(dk, &tm_k, &bars.full[s], 0, j * BN, (int)hk, (int)b);
        tma_load_4d(dk + BOX, &tm_k, &bars.full[s], 64, j * BN, (int)hk, (int)b);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ================================================================ MMA issuer + reducer
    if (lane == 0) {
      mbar_wait(&bars.q_full, 0);
      tc_fence_after();
      auto issue_s = [&](int j) {
        const int s = j % NST;
        mbar_wait(&bars.full[s], (uint32_t)(j / NST) & 1u);
        tc_fence_after();
        const uint32_t sk = base + SMEM_K + s * TILE;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * BOX + (kk & 3) * 32;
          mma_ts(tmem + ((j & 1) ? 128u : 0u), tmem + Q_COL + kk * 8, make_desc(sk + off, 16, 1024), IDESC_S, kk > 0 ? 1u : 0u);
        }
        mma_commit(&bars.s_full[j & 1]);
        mma_commit(&bars.empty[s]);  // the K stage is free once S_j has read it
      };
      issue_s(0);
      const float inv_n = 1.f / (float)nrows;
      float captured = 0.f;
      float *mh = a.m_hat + (bh * a.nq + gq) * a.nk;
      for (int j = 0; j < cnt; ++j) {
        if (j + 1 < cnt) issue_s(j + 1);
        mbar_wait(&bars.p_full[j & 1], (uint32_t)(j >> 1) & 1u);  // the 8 partials of tile j are in smem
        if constexpr (kMass) {
          const volatile float *pj = part + (j & 1) * 8;
          float tot = 0.f;
#pragma unroll
          for (int w = 0; w < 8; ++w) tot += pj[w];
          const float mj = tot * inv_n;
          mh[j] = mj;  // (consumes the smem reads before S_{j+2} can be issued)
          if ((sel[j >> 5] >> (j & 31)) & 1u) captured += mj;
        }
        if constexpr (kExt) {
          const volatile float *px = part + 16 + (j & 1) * 8, *pn = part + 32 + (j & 1) * 8;
          float mx = -INFINITY, mn = INFINITY;
#pragma unroll
          for (int w = 0; w < 8; ++w) { mx = fmaxf(mx, px[w]); mn = fminf(mn, pn[w]); }
          a.s_max[(bh * a.nq + gq) * a.nk + j] = mx;
          a.s_min[(bh * a.nq + gq) * a.nk + j] = mn;
        }
      }
      if (kMass && a.captured) a.captured[bh * a.nq + gq] = captured;
    }
    __syncwarp();
  } else {
    // ================================================================ mass warps
    const int sw = warp - 2;     // 0..7
    const int hf = sw >> 2;      // column half
    const int qd = warp & 3;     // TMEM lane quadrant
    const int r = qd * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(qd * 32) << 16);
    {  // Q row half -> TMEM (A operand of S = Q K^T)
      uint32_t qv[32];
      const __nv_bfloat16 *qp = static_cast<const __nv_bfloat16 *>(a.q) + b * a.qs[0] + h * a.qs[1] + (row0 + r) * a.qs[2] + hf * 64;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint4 u = r < nrows ? ldg16(qp + 8 * i) : make_uint4(0, 0, 0, 0);
        qv[4 * i] = u.x; qv[4 * i + 1] = u.y; qv[4 * i + 2] = u.z; qv[4 * i + 3] = u.w;
      }
      tmem_st_x32(trow + Q_COL + hf * 32, qv);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.q_full);
    }
    const float c = a.scale * 1.4426950408889634f;
    float nl = -INFINITY;  // rows past L add 0
    if constexpr (kMass) nl = r < nrows ? -a.lse[bh * a.lq + row0 + r] * 1.4426950408889634f : -INFINITY;
    const int64_t ragged_valid = a.lk - (a.nk - 1) * (int64_t)BN;
    for (int j = 0; j < cnt; ++j) {
      mbar_wait(&bars.s_full[j & 1], (uint32_t)(j >> 1) & 1u);
      tc_fence_after();
      uint32_t sr[64];
      tmem_ld_x32(trow + ((j & 1) ? 128u : 0u) + hf * 64, sr);
      tmem_ld_x32(trow + ((j & 1) ? 128u : 0u) + hf * 64 + 32, sr + 32);
      tmem_wait_ld();
      const int valid = j == cnt - 1 ? (int)ragged_valid - hf * 64 : 64;  // key columns inside the sequence
      if constexpr (kMass) {
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          const float p = ex2(fmaf(__uint_as_float(sr[i]), c, nl));
          acc += i < valid ? p : 0.f;
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) part[(j & 1) * 8 + sw] = acc;
      }
      if constexpr (kExt) {  // token-logit extremes over the valid rows and columns of the block pair
        float mx = -INFINITY, mn = INFINITY;
        if (r < nrows) {
#pragma unroll
          for (int i = 0; i < 64; ++i) {
            const float x = __uint_as_float(sr[i]);
            if (i < valid) { mx = fmaxf(mx, x); mn = fminf(mn, x); }
          }
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) {
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
          mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, off));
        }
        if (lane == 0) { part[16 + (j & 1) * 8 + sw] = mx; part[32 + (j & 1) * 8 + sw] = mn; }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.p_full[j & 1]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

}  // namespace mass
}  // namespace sm100

bool block_mass_supported(const MassArgs &a) { return a.d == 128 && a.B == 128 && a.nk <= 32 * sm100::mass::kMaskWords; }

namespace {
template <bool kMass, bool kExt>
cudaError_t launch_mass_variant(const MassArgs &a, const CUtensorMap &mk, cudaStream_t st) {
  using namespace sm100::mass;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(block_mass_kernel<kMass, kExt>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((unsigned)a.nq, (unsigned)(a.batch * a.hq));
  block_mass_kernel<kMass, kExt><<<grid, kThreads, SMEM_BYTES, st>>>(a, mk);
  return cudaGetLastError();
}
}  // namespace

// m_hat (a.m_hat, needs a.lse) and / or the token-logit extremes (a.s_max / a.s_min)
cudaError_t launch_block_mass(const MassArgs &a, cudaStream_t st) {
  using namespace sm100;
  CUtensorMap mk;
  if (!get_encode()) return cudaErrorNotSupported;
  if (!make_map(&mk, a.k, a.batch, a.hkv, a.lk, a.d, a.ks, 128)) return cudaErrorInvalidValue;
  const bool mass = a.m_hat != nullptr, ext = a.s_max != nullptr;
  if (mass && ext) return launch_mass_variant<true, true>(a, mk, st);
  if (mass) return launch_mass_variant<true, false>(a, mk, st);
  if (ext) return launch_mass_variant<false, true>(a, mk, st);
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------ Eq. logits-bound
// R_g = max_{i in I(g)} ||x_i - xbar_g||_2 (radius) and M_g = max_{i in I(g)} ||x_i||_2 (max norm)
// per block of the sorted copy x [b, H, L, D] (contiguous), in fp64 against the fp64 block means.
// One CTA (4 warps) per (block, b*H); a warp per row, lane owns D/32 features.
template <typename T, int D>
__global__ void __launch_bounds__(128) block_radius_kernel(const T *__restrict__ x, const double *__restrict__ mean,
                                                          int64_t L, int B, int64_t n_blk, double *__restrict__ R,
                                                          double *__restrict__ M) {
  constexpr int E = D / 32;
  const int64_t g = blockIdx.x, bh = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = g * B, nr = imin64(B, L - r0);
  double mu[E];
#pragma unroll
  for (int e = 0; e < E; ++e) mu[e] = mean[(bh * n_blk + g) * D + lane * E + e];
  double rmax = 0.0, mmax = 0.0;  // squared
  for (int64_t i = warp; i < nr; i += 4) {
    const T *row = x + (bh * L + r0 + i) * D + lane * E;
    double r2 = 0.0, m2 = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const double v = (double)to_float(row[e]);
      const double dv = v - mu[e];
      r2 = fma(dv, dv, r2);
      m2 = fma(v, v, m2);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      r2 += __shfl_xor_sync(0xffffffffu, r2, off);
      m2 += __shfl_xor_sync(0xffffffffu, m2, off);
    }
    rmax = fmax(rmax, r2);
    mmax = fmax(mmax, m2);
  }
  __shared__ double sr[4], sm[4];
  if (lane == 0) { sr[warp] = rmax; sm[warp] = mmax; }
  __syncthreads();
  if (threadIdx.x == 0) {
    R[bh * n_blk + g] = sqrt(fmax(fmax(sr[0], sr[1]), fmax(sr[2], sr[3])));
    M[bh * n_blk + g] = sqrt(fmax(fmax(sm[0], sm[1]), fmax(sm[2], sm[3])));
  }
}

// U[g_q, g_k] = (R^Q M^K + M^Q R^K + R^Q R^K) / sqrt(d) (Eq. logits-bound) and the observed
// max |l_hat - l| = max(S_max/sqrt(d) - l, l - S_min/sqrt(d)) with l = Qbar.Kbar/sqrt(d) (fp64).
__global__ void deviation_finalize_kernel(int64_t hq, int64_t grp, int64_t nq, int64_t nk, const double *__restrict__ rq,
                                          const double *__restrict__ mq, const double *__restrict__ rk,
                                          const double *__restrict__ mk, const double *__restrict__ logit,
                                          const float *__restrict__ smax, const float *__restrict__ smin,
                                          double inv_sqrt_d, double *__restrict__ U, double *__restrict__ dev,
                                          int64_t total) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gk = e % nk, row = e / nk;  // row = (b*hq + h)*nq + gq
    const int64_t bhq = row / nq, b = bhq / hq, h = bhq - b * hq;
    const int64_t kidx = (b * (hq / grp) + h / grp) * nk + gk;
    const double Rq = rq[row], Mq = mq[row], Rk = rk[kidx], Mk = mk[kidx];
    if (U) U[e] = (Rq * Mk + Mq * Rk + Rq * Rk) * inv_sqrt_d;
    if (dev) {
      const double l = logit[e];
      dev[e] = fmax((double)smax[e] * inv_sqrt_d - l, l - (double)smin[e] * inv_sqrt_d);
    }
  }
}

cudaError_t launch_block_radius(int dtype, int d, const void *x, int64_t batch_heads, int64_t L, int B,
                                const double *mean, double *R, double *M, cudaStream_t st) {
  const int64_t n_blk = (L + B - 1) / B;
  dim3 grid((unsigned)n_blk, (unsigned)batch_heads);
  if (dtype == 0 && d == 128) block_radius_kernel<__nv_bfloat16, 128><<<grid, 128, 0, st>>>(static_cast<const __nv_bfloat16 *>(x), mean, L, B, n_blk, R, M);
  else if (dtype == 0) block_radius_kernel<__nv_bfloat16, 64><<<grid, 128, 0, st>>>(static_cast<const __nv_bfloat16 *>(x), mean, L, B, n_blk, R, M);
  else if (d == 128) block_radius_kernel<float, 128><<<grid, 128, 0, st>>>(static_cast<const float *>(x), mean, L, B, n_blk, R, M);
  else block_radius_kernel<float, 64><<<grid, 128, 0, st>>>(static_cast<const float *>(x), mean, L, B, n_blk, R, M);
  return cudaGetLastError();
}

cudaError_t launch_deviation_finalize(int64_t batch, int64_t hq, int64_t hkv, int64_t nq, int64_t nk, const double *rq,
                                      const double *mq, const double *rk, const double *mk, const double *logit,
                                      const float *smax, const float *smin, double inv_sqrt_d, double *U, double *dev,
                                      cudaStream_t st) {
  const int64_t total = batch * hq * nq * nk;
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
  deviation_finalize_kernel<<<grid, 256, 0, st>>>(hq, hq / hkv, nq, nk, rq, mq, rk, mk, logit, smax, smin, inv_sqrt_d, U,
                                                  dev, total);
  return cudaGetLastError();
}

}  // namespace baatt
