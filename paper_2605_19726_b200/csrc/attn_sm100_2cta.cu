// attn_sm100_2cta.cu — K5 for B = 128 on a 2-CTA cluster (tcgen05 cta_group::2).
//
// Same computation as attn_sm100.cu (Alg. 1 steps 11-12, PAPER.md P:563-566:
// non-causal attention of each query block over its selected key blocks only,
// P:263-264, rows written back to pi_q(i)), but the two CTAs of a
// cluster own ADJACENT query blocks 2p and 2p+1 of one head and walk the union
// of their two index lists.  Norm-sorted neighbours select nearly the same key
// blocks, so every key/value tile is fetched once for both.
//
// Per union tile u, CTA r (r = cluster rank) loads only
//   K_u rows [64r, 64r + 64)    (the N-half of B = K^T for S = Q K^T), and
//   V_u cols [64r, 64r + 64)    (the N-half of B = V   for O += P V),
// i.e. 32 KB instead of 64 KB, and the leader issues tcgen05.mma.cta_group::2
// with M = 256: rows 0-127 are the leader's query block (Q and P in its TMEM),
// rows 128-255 the peer's.  Rows of a block that did not select u get P = 0.
//
// Q (each CTA's 128 rows) sits in smem; S = Q K^T is an SS-form M = 256 MMA
// into a triple-buffered TMEM accumulator issued two tiles ahead of the PV that
// waits for the softmax (TMEM: S0 S1 S2 O = 512 columns).
// Synchronisation: the leader owns the "full" barriers (q_full / k_full /
// v_full get the TMA bytes of both CTAs and one arrive per producer; p_full
// gets one arrive per softmax warp of both CTAs, the peer's through mapa);
// every "empty" barrier and s_full / o_done exist in both CTAs and are
// signalled by multicast tcgen05.commit.  Warp roles otherwise as in
// attn_sm100.cu.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"
#include "sm100_ptx.cuh"

namespace baatt {
namespace sm100 {

namespace pair2 {

constexpr int BM = 128;                          // query rows per CTA (one query block)
constexpr int BN = 128;                          // key rows per tile (one key block)
constexpr int HD = 128;
constexpr uint32_t O_COL = 384;
constexpr int NSB = 3;                           // S/P buffers: S_{j+2} queued before PV_j
constexpr int kSoftmaxWarp0 = 2;
constexpr int kVProducerWarp = 10;
constexpr int kThreads = 352;
constexpr float kRescaleThreshold = 8.0f;
constexpr int kMaskWords = 1024;
constexpr uint32_t K_BOX = 64 * 64 * 2;          // 64 key rows x 64 d-cols
constexpr uint32_t K_HALF = 2 * K_BOX;           // this CTA's 64 key rows x 128 d (16 KB)
constexpr uint32_t V_HALF = 128 * 64 * 2;        // 128 key rows x this CTA's 64 d-cols (16 KB)
constexpr uint32_t Q_BOX = 128 * 64 * 2;         // this CTA's 128 query rows x 64 d-cols
constexpr uint32_t Q_BYTES = 2 * Q_BOX;
constexpr int NKS = 6;
constexpr int NVS = 4;
// kind::f16, D fp32, A/B bf16, M = 256 (cta_group::2), N = 128
constexpr uint32_t IDESC_S = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
constexpr uint32_t IDESC_O = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(HD >> 3) << 17) | ((uint32_t)(256 >> 4) << 24) |
                             (1u << 16);  // B = V MN-major
constexpr uint32_t SMEM_Q = 0;
constexpr uint32_t SMEM_K = Q_BYTES;
constexpr uint32_t SMEM_V = SMEM_K + NKS * K_HALF;
constexpr uint32_t SMEM_RED = SMEM_V + NVS * V_HALF;
constexpr uint32_t SMEM_RED2 = SMEM_RED + 2 * 2 * 128 * 4;
constexpr uint32_t SMEM_MASK = SMEM_RED2 + 2 * 128 * 4;
constexpr uint32_t SMEM_BARS = SMEM_MASK + 2 * kMaskWords * 4;
constexpr uint32_t SMEM_BYTES = SMEM_BARS + 512 + 1024;
BA_DEVICE constexpr uint32_t s_col(int buf) { return (uint32_t)(buf * 128); }

struct __align__(8) Bars {
  uint64_t q_full;                    // leader: 2 arrivals + both CTAs' Q bytes
  uint64_t k_full[NKS], k_empty[NKS];  // full: leader (2 arrivals + bytes); empty: both (multicast commit)
  uint64_t v_full[NVS], v_empty[NVS];
  uint64_t s_full[NSB], p_full[NSB];  // s_full: both (commit); p_full: leader (16 arrivals)
  uint64_t o_done[NSB];               // both (commit)
  uint64_t o_final;                   // both (commit), single phase: every PV of the tile completed
  uint32_t tmem_base;
  uint32_t n_union;
  uint32_t last_ragged;
};

struct UnionWalk {
  const uint32_t *ma, *mb;
  int w;
  uint32_t rem;
  BA_DEVICE void init(const uint32_t *a_, const uint32_t *b_) { ma = a_; mb = b_; w = 0; rem = a_[0] | b_[0]; }
  BA_DEVICE int next() {
    while (rem == 0) { ++w; rem = ma[w] | mb[w]; }
    const int bit = __ffs(rem) - 1;
    rem &= rem - 1;
    return w * 32 + bit;
  }
};

constexpr int kTraceTiles = 10;
template <bool kTrace, int kEmu = 0, bool kNoSoftmax = false>
__global__ void __launch_bounds__(kThreads, 1)
attn_2cta_kernel(const AttnArgs a, const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                 const __grid_constant__ CUtensorMap tm_v) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t *smem = smem_raw + (base - raw);
  Bars &bars = *reinterpret_cast<Bars *>(smem + SMEM_BARS);
  float *red = reinterpret_cast<float *>(smem + SMEM_RED);
  float *red2 = reinterpret_cast<float *>(smem + SMEM_RED2);
  uint32_t *mask_a = reinterpret_cast<uint32_t *>(smem + SMEM_MASK);
  uint32_t *mask_b = mask_a + kMaskWords;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1;
  const int64_t bh = blockIdx.y;
  const int64_t b = bh / a.hq, h = bh - b * a.hq;
  const int64_t hk = h / (a.hq / a.hkv);
  const int nw = (int)((a.nk + 31) >> 5);
  __shared__ long long trace[12][kTraceTiles];
  const bool tr = kTrace && blockIdx.x < 2 && blockIdx.y == 0;
  const long long t_origin = kTrace ? clock64() : 0;
#define TR(slot, j) do { if (tr && (j) < kTraceTiles) trace[slot][j] = clock64() - t_origin; } while (0)

  // ---- key-block sets of both query blocks of the pair (both CTAs build both)
  const int64_t ga = 2 * (int64_t)pair;
  const bool has_b = ga + 1 < a.nq;
  for (int w = threadIdx.x; w < 2 * kMaskWords; w += kThreads) mask_a[w] = 0u;
  __syncthreads();
  for (int q2 = 0; q2 < (has_b ? 2 : 1); ++q2) {
    const int64_t row = bh * a.nq + ga + q2;
    uint32_t *m = q2 ? mask_b : mask_a;
    if (a.kv_index) {
      const int cnt = a.kv_count ? a.kv_count[row] : (int)a.kv_stride;
      const int32_t *idx = a.kv_index + row * a.kv_stride;
      for (int e = threadIdx.x; e < cnt; e += kThreads) {
        const int g = idx[e];
        atomicOr(&m[g >> 5], 1u << (g & 31));
      }
    } else {
      for (int w = threadIdx.x; w < nw; w += kThreads)
        m[w] = (w + 1) * 32 <= a.nk ? 0xffffffffu : ((1u << (a.nk & 31)) - 1u);
    }
  }
  __syncthreads();
  if (warp == 0) {
    unsigned c = 0;
    for (int w = lane; w < nw; w += 32) c += __popc(mask_a[w] | mask_b[w]);
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) {
      bars.n_union = c;
      const int64_t gl = a.nk - 1;
      const bool sel_last = ((mask_a[gl >> 5] | mask_b[gl >> 5]) >> (gl & 31)) & 1u;
      bars.last_ragged = sel_last && (a.lk - gl * (int64_t)BN) < BN;
    }
  }
  if (warp == 0 && lane == 0) {
    mbar_init(&bars.q_full, 2);
    for (int s = 0; s < NKS; ++s) { mbar_init(&bars.k_full[s], 2); mbar_init(&bars.k_empty[s], 1); }
    for (int s = 0; s < NVS; ++s) { mbar_init(&bars.v_full[s], 2); mbar_init(&bars.v_empty[s], 1); }
    for (int s = 0; s < NSB; ++s) {
      mbar_init(&bars.s_full[s], 1);
      mbar_init(&bars.p_full[s], 16);
      mbar_init(&bars.o_done[s], 1);
    }
    mbar_init(&bars.o_final, 1);
    fence_barrier_init();
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
  }
  if (warp == 1) {  // same warp in both CTAs: paired allocation
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&bars.tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();  // barrier inits and TMEM allocation visible to the peer
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;
  const int cnt = (int)bars.n_union;
  const bool last_ragged = bars.last_ragged != 0u;

  if (warp == 0 || warp == kVProducerWarp) {
    // ================================================================ TMA producers (both CTAs)
    const bool is_k = warp == 0;
    const int nst = is_k ? NKS : NVS;
    uint64_t *full = is_k ? bars.k_full : bars.v_full;
    uint64_t *empty = is_k ? bars.k_empty : bars.v_empty;
    const uint32_t ring = base + (is_k ? SMEM_K : SMEM_V);
    const uint32_t half_bytes = is_k ? K_HALF : V_HALF;
    if (lane == 0 && cnt > 0) {
      if (is_k) {  // this CTA's 128 query rows, bytes counted on the leader's q_full
        const uint32_t qbar0 = map_to_rank(smem_u32(&bars.q_full), 0);
        if (leader) mbar_expect_tx(&bars.q_full, 2 * Q_BYTES);
        tma_load_4d_2sm(base + SMEM_Q, &tm_q, qbar0, 0, (int)((ga + rank) * BM), (int)h, (int)b);
        tma_load_4d_2sm(base + SMEM_Q + Q_BOX, &tm_q, qbar0, 64, (int)((ga + rank) * BM), (int)h, (int)b);
        if (!leader) mbar_arrive_remote(qbar0);
      }
      UnionWalk walk;
      walk.init(mask_a, mask_b);
      for (int j = 0; j < cnt; ++j) {
        const int gk = walk.next();
        const int s = j % nst;
        const uint32_t ph = (uint32_t)(j / nst) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        TR(is_k ? 0 : 1, j);
        const uint32_t mbar0 = map_to_rank(smem_u32(&full[s]), 0);
        const uint32_t dst = ring + s * half_bytes;
        if (leader) mbar_expect_tx(&full[s], 2 * half_bytes);  // both halves land on the leader's barrier
        if (is_k) {  // rows [gk*128 + 64r, +64), both 64-column boxes
          tma_load_4d_2sm(dst, &tm_k, mbar0, 0, gk * BN + 64 * (int)rank, (int)hk, (int)b);
          tma_load_4d_2sm(dst + K_BOX, &tm_k, mbar0, 64, gk * BN + 64 * (int)rank, (int)hk, (int)b);
        } else {     // rows [gk*128, +128), columns [64r, +64)
          tma_load_4d_2sm(dst, &tm_v, mbar0, 64 * (int)rank, gk * BN, (int)hk, (int)b);
        }
        if (!leader) mbar_arrive_remote(mbar0);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ================================================================ MMA issuer (leader only)
    if (leader && lane == 0 && cnt > 0) {
      mbar_wait(&bars.q_full, 0);
      tc_fence_after();
      auto issue_s = [&](int j) {
        const int s = j % NKS;
        mbar_wait(&bars.k_full[s], (uint32_t)(j / NKS) & 1u);
        TR(2, j);
        tc_fence_after();
        const uint32_t sk = base + SMEM_K + s * K_HALF;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          mma_ss_2sm(tmem + s_col(j % NSB), make_desc(base + SMEM_Q + (kk >> 2) * Q_BOX + (kk & 3) * 32, 16, 1024),
                     make_desc(sk + (kk >> 2) * K_BOX + (kk & 3) * 32, 16, 1024), IDESC_S, kk > 0 ? 1u : 0u);
        mma_commit_2sm_mc(&bars.k_empty[s], 0x3);
        mma_commit_2sm_mc(&bars.s_full[j % NSB], 0x3);
      };
      issue_s(0);
      if (cnt > 1) issue_s(1);
      for (int j = 0; j < cnt; ++j) {
        if (j + 2 < cnt) issue_s(j + 2);
        mbar_wait(&bars.p_full[j % NSB], (uint32_t)(j / NSB) & 1u);
        TR(3, j);
        const int s = j % NVS;
        mbar_wait(&bars.v_full[s], (uint32_t)(j / NVS) & 1u);
        TR(4, j);
        tc_fence_after();
        const uint32_t sv = base + SMEM_V + s * V_HALF;
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)
          mma_ts_2sm(tmem + O_COL, tmem + s_col(j % NSB) + kk * 8, make_desc(sv + kk * 2048, V_HALF, 1024), IDESC_O,
                     (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit_2sm_mc(&bars.v_empty[s], 0x3);
        mma_commit_2sm_mc(&bars.o_done[j % NSB], 0x3);
      }
      mma_commit_2sm_mc(&bars.o_final, 0x3);
    }
    __syncwarp();
  } else if (warp >= kSoftmaxWarp0 && warp < kSoftmaxWarp0 + 8) {
    // ================================================================ softmax + epilogue (both CTAs)
    constexpr int HC = 64;
    const int sw = warp - kSoftmaxWarp0;
    const int hf = sw >> 2;
    const int qd = warp & 3;
    const int r = qd * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(qd * 32) << 16);
    const int64_t row0 = (ga + rank) * (int64_t)BM;
    const int nrows = (int)imin64(BM, imin64(a.lq - row0, BM));
    const uint32_t *my_mask = rank ? mask_b : mask_a;
    uint32_t p_full0[NSB];
#pragma unroll
    for (int i = 0; i < NSB; ++i) p_full0[i] = map_to_rank(smem_u32(&bars.p_full[i]), 0);
    const float c = a.scale * 1.4426950408889634f;
    const int64_t ragged_valid = a.lk - (a.nk - 1) * (int64_t)BN;
    float m = -INFINITY, l = 0.f;
    uint32_t sr[HC];
    UnionWalk walk;
    walk.init(mask_a, mask_b);
    for (int j = 0; j < cnt; ++j) {
      const int gk = walk.next();
      const bool mine = (my_mask[gk >> 5] >> (gk & 31)) & 1u;  // CTA-uniform
      mbar_wait(&bars.s_full[j % NSB], (uint32_t)(j / NSB) & 1u);
      if (lane == 0 && qd == 0 && hf == 0) TR(5, j);
      tc_fence_after();
      if constexpr (kNoSoftmax) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(p_full0[j % NSB]);
        continue;
      }
      if (mine) {
        tmem_ld_x32(trow + s_col(j % NSB) + hf * HC, sr);
        tmem_ld_x32(trow + s_col(j % NSB) + hf * HC + 32, sr + 32);
        tmem_wait_ld();
        if (last_ragged && j == cnt - 1) {
#pragma unroll
          for (int i = 0; i < HC; ++i)
            if (hf * HC + i >= ragged_valid) sr[i] = __float_as_uint(-INFINITY);
        }
      }
      float pmax = -INFINITY;
      if (mine) {
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int i = 0; i < HC; i += 8) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            m4[u] = fmax3(m4[u], __uint_as_float(sr[i + 2 * u]), __uint_as_float(sr[i + 2 * u + 1]));
        }
        pmax = fmaxf(fmax3(m4[0], m4[1], m4[2]), m4[3]);
      }
      red[((j & 1) * 2 + hf) * 128 + r] = pmax;
      tc_fence_before();
      named_bar_sync(1 + qd, 64);
      tc_fence_after();
      if (lane == 0 && qd == 0 && hf == 0) TR(6, j);
      if (mine) {
        const float mt = fmaxf(pmax, red[((j & 1) * 2 + (hf ^ 1)) * 128 + r]) * c;
        if (m == -INFINITY) {
          m = mt;
        } else {
          const bool need = mt > m + kRescaleThreshold;
          if (__any_sync(0xffffffffu, need)) {
            float corr = 1.f;
            if (need) { corr = ex2(m - mt); m = mt; }
            mbar_wait(&bars.o_done[(j - 1) % NSB], (uint32_t)((j - 1) / NSB) & 1u);
            tc_fence_after();
            uint32_t ov[16];
#pragma unroll
            for (int q2 = 0; q2 < 4; ++q2) {
              tmem_ld_x16(trow + O_COL + hf * 64 + q2 * 16, ov);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 16; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * corr);
              tmem_st_x16(trow + O_COL + hf * 64 + q2 * 16, ov);
            }
            l *= corr;
          }
        }
        const uint64_t c2 = f2(c, c), nm2 = f2(-m, -m);
        uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
        for (int i = 0; i < HC / 2; ++i) {
          const uint64_t x2 = ffma2(f2(__uint_as_float(sr[2 * i]), __uint_as_float(sr[2 * i + 1])), c2, nm2);
          uint64_t p2;
          if ((i & 7) < kEmu) {
            p2 = exp2_poly2(x2);
          } else {
            float x0, x1;
            unf2(x2, x0, x1);
            p2 = f2(ex2(x0), ex2(x1));
          }
          acc2[i & 3] = fadd2(acc2[i & 3], p2);
          float p0, p1;
          unf2(p2, p0, p1);
          sr[i] = pack_bf16(p0, p1);
        }
        const uint64_t t2 = fadd2(fadd2(acc2[0], acc2[1]), fadd2(acc2[2], acc2[3]));
        float a0, a1;
        unf2(t2, a0, a1);
        l += a0 + a1;
      } else {
#pragma unroll
        for (int i = 0; i < HC / 2; ++i) sr[i] = 0u;
      }
      if (lane == 0 && qd == 0 && hf == 0) TR(7, j);
      tmem_st_x32(trow + s_col(j % NSB) + hf * (HC / 2), sr);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(p_full0[j % NSB]);
      if (lane == 0 && qd == 0 && hf == 0) TR(8, j);
    }
    red2[hf * 128 + r] = l;
    named_bar_sync(1 + qd, 64);
    const float lt = l + red2[(hf ^ 1) * 128 + r];
    if (cnt > 0) {
      // not o_done: when this tile's softmax skipped its last tiles it can arrive here with
      // only cnt-2 PVs complete, which the parity of o_done cannot tell from cnt
      mbar_wait(&bars.o_final, 0);
      tc_fence_after();
    }
    const float inv = lt > 0.f ? 1.f / lt : 0.f;
    int64_t orow = row0 + r;
    if (r < nrows && a.perm_q) orow = a.perm_q[bh * a.lq + row0 + r];
    __nv_bfloat16 *o = static_cast<__nv_bfloat16 *>(a.out) + b * a.os[0] + h * a.os[1] + orow * a.os[2] + hf * 64;
#pragma unroll
    for (int q2 = 0; q2 < 2; ++q2) {
      uint32_t ov[32];
      tmem_ld_x32(trow + O_COL + hf * 64 + q2 * 32, ov);
      tmem_wait_ld();
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)
        pk[i] = pack_bf16(__uint_as_float(ov[2 * i]) * inv, __uint_as_float(ov[2 * i + 1]) * inv);
      if (r < nrows) {
        uint4 *dst = reinterpret_cast<uint4 *>(o + q2 * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
      }
    }
    if (a.lse && hf == 0 && r < nrows) a.lse[bh * a.lq + orow] = lt > 0.f ? (m + log2f(lt)) * 0.69314718055994531f : -INFINITY;
  }
  tc_fence_before();
  __syncthreads();
  if (tr && threadIdx.x == 0) {
    const char *names[9] = {"prod_K", "prod_V", "mma_S", "mma_pwait", "mma_PV", "sm_wait", "sm_bar", "sm_exp", "sm_arr"};
    for (int k = 0; k < 9; ++k) {
      printf("TRACE r%u %-9s", rank, names[k]);
      for (int j = 0; j < kTraceTiles && j < cnt; ++j) printf(" %7lld", trace[k][j]);
      printf("\n");
    }
  }
#undef TR
  cluster_sync();  // the leader's MMAs wrote the peer's TMEM: both finish before either frees it
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

}  // namespace pair2

bool make_map(CUtensorMap *m, const void *ptr, int64_t b, int64_t H, int64_t L, int64_t d, const int64_t *s, int rows);
PFN_cuTensorMapEncodeTiled_v12000 get_encode();

}  // namespace sm100

bool attn_2cta_supported(const AttnArgs &a) {
  return a.dtype == 0 && a.d == 128 && a.B == 128 && a.nk <= 32 * sm100::pair2::kMaskWords;
}

cudaError_t launch_attn_2cta(const AttnArgs &a, cudaStream_t st) {
  using namespace sm100;
  using namespace sm100::pair2;
  CUtensorMap mq, mk, mv;
  if (!get_encode()) return cudaErrorNotSupported;
  if (!make_map(&mq, a.q, a.batch, a.hq, a.lq, a.d, a.qs, 128) || !make_map(&mk, a.k, a.batch, a.hkv, a.lk, a.d, a.ks, 64) ||
      !make_map(&mv, a.v, a.batch, a.hkv, a.lk, a.d, a.vs, 128))
    return cudaErrorInvalidValue;
  static int dbg = -1, emu = 0;
  if (dbg < 0) {
    const char *d = getenv("BA_ATTN_DEBUG");
    dbg = d ? atoi(d) : 0;
    const char *e = getenv("BA_EXP_EMU");
    emu = e ? atoi(e) : 0;
    void (*ks[5])(const AttnArgs, const CUtensorMap, const CUtensorMap, const CUtensorMap) = {
        attn_2cta_kernel<false, 0, false>, attn_2cta_kernel<true, 0, false>, attn_2cta_kernel<false, 0, true>,
        attn_2cta_kernel<false, 1, false>, attn_2cta_kernel<false, 2, false>};
    for (auto k : ks) {
      cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES);
      if (err != cudaSuccess) return err;
    }
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(2 * ((a.nq + 1) / 2)), (unsigned)(a.batch * a.hq));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 2;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  if (dbg == 2) return cudaLaunchKernelEx(&cfg, attn_2cta_kernel<true, 0, false>, a, mq, mk, mv);
  if (dbg == 1) return cudaLaunchKernelEx(&cfg, attn_2cta_kernel<false, 0, true>, a, mq, mk, mv);
  if (emu == 1) return cudaLaunchKernelEx(&cfg, attn_2cta_kernel<false, 1, false>, a, mq, mk, mv);
  if (emu == 2) return cudaLaunchKernelEx(&cfg, attn_2cta_kernel<false, 2, false>, a, mq, mk, mv);
  return cudaLaunchKernelEx(&cfg, attn_2cta_kernel<false, 0, false>, a, mq, mk, mv);
}

}  // namespace baatt
