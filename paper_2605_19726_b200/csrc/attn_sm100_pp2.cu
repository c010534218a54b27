// attn_sm100_pp2.cu — K5 for B = 128 on a 2-CTA cluster: the ping-pong pair
// kernel (attn_sm100_pp.cu) with every MMA issued as tcgen05.mma.cta_group::2
// (M = 256) over the two SMs of the cluster (tcgen05 + TMEM + TMA, sm_100a).
//
// Computes Alg. 1 steps 11-12: each query block attends
// over its selected key blocks only, online softmax, rows
// written back to pi_q(i).  Non-causal.
//
// A cluster owns a QUAD of adjacent query blocks 4q .. 4q+3 of one head (their
// norm-sorted neighbourhoods select nearly the same key blocks: the union of the
// four lists is 1.017 kappa at A and 1.019 kappa at C, measured) and walks the
// union of their lists.  CTA r holds blocks 4q + 2x + r for x = 0, 1; MMA "x"
// covers rows of block 4q+2x (CTA 0, TMEM lanes of SM 0) and 4q+2x+1 (CTA 1).
// Every K/V tile is fetched once for the four blocks and split between the
// SMs: CTA r loads keys [64r, 64r+64) of K_u (its N-half of B = K^T for
// S = Q K^T) and the columns [64r, 64r+64) of V_u (its N-half of B = V for
// O += P V).  Per SM and union tile that is 160 KB of shared-memory operand +
// TMA traffic for 2048 tensor cycles (78 B/clk), against 256 KB (125 B/clk,
// the port's limit) for the single-CTA pair kernel.
//
// Warps (both CTAs): 0-3 softmax of block x = 0, 4-7 softmax of block x = 1 (one
//        thread per row, 128 columns), 8 TMA producer (own Q blocks, own
//        halves of K_u / V_u into an 8-slot ring of 16 KB), 9 TMEM owner and,
//        in CTA 0 only, the single MMA issuer; 10-11 idle.
// TMEM (each CTA, its 128 rows): S_0 [0,128), S_1 [128,256), O_0 [256,384),
// O_1 [384,512).  Issue order per union tile u (as the pair kernel):
//   PV_0(u-1) | S_0(u) | PV_1(u-1) | S_1(u)
// Barriers: the "full" ones (q_full, full[s]) and p_part live in CTA 0 (both
// CTAs' TMA bytes and softmax arrivals land there); empty[s], s_full and
// o_final exist in both CTAs and are signalled by multicast tcgen05.commit.
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

bool make_map(CUtensorMap *m, const void *ptr, int64_t b, int64_t H, int64_t L, int64_t d, const int64_t *s, int rows);
PFN_cuTensorMapEncodeTiled_v12000 get_encode();

namespace pp2 {

constexpr int BM = 128, BN = 128, HD = 128;
constexpr uint32_t QBOX = 128 * 64 * 2;      // 128 rows x 64 bf16 columns (16 KB)
constexpr uint32_t QTILE = 2 * QBOX;         // one query block, 128 x 128 (32 KB)
constexpr uint32_t KBOX = 64 * 64 * 2;       // 64 key rows x 64 columns (8 KB)
constexpr uint32_t HALF = 16 * 1024;         // a K half (64 keys x 128) or a V half (128 keys x 64 cols)
// Ring of 16 KB half-tile slots filled K_0, V_0, K_1, V_1, ...; a slot is released by a
// (multicast) commit after its last reader: K_u after S_1(u), V_u after PV_1(u).
constexpr int NSLOT = 8;
BA_DEVICE constexpr uint32_t s_col(int x) { return x ? 128u : 0u; }
constexpr uint32_t O_COL0 = 256;
constexpr int kProducerWarp = 8, kMmaWarp = 9;
constexpr int kPSplit = 2;                   // P handed to the MMA in two key halves (as the pair kernel)
constexpr int kThreads = 384;
constexpr int kRegsSoftmax = 208, kRegsSide = 80;
constexpr float kRescaleThreshold = 8.0f;
constexpr int kMaskWords = 256;              // nk <= 8192
constexpr int kDefaultEmu = 1;
constexpr uint32_t SMEM_Q = 0;                                  // Q_0, Q_1 (this CTA's two blocks)
constexpr uint32_t SMEM_SLOT = 2 * QTILE;
constexpr uint32_t SMEM_MASK = SMEM_SLOT + NSLOT * HALF;        // uint32 [4][kMaskWords]
constexpr uint32_t SMEM_BARS = SMEM_MASK + 4 * kMaskWords * 4;
constexpr uint32_t SMEM_BYTES = SMEM_BARS + 256;
static_assert(SMEM_BYTES <= 232448, "exceeds the 227 KB opt-in shared memory");
// kind::f16, D fp32, A/B bf16, M = 256 (cta_group::2), N = 128
constexpr uint32_t IDESC_S = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
constexpr uint32_t IDESC_O = IDESC_S | (1u << 16);  // B = V MN-major (N = d = 128)

struct __align__(8) Bars {
  uint64_t q_full;                                  // CTA 0: 2 arrivals + both CTAs' Q bytes
  uint64_t full[NSLOT], empty[NSLOT];               // full: CTA 0 (2 arrivals + bytes); empty: both
  uint64_t s_full[2], p_part[2][kPSplit];           // s_full: both; p_part: CTA 0 (8 warp arrivals)
  uint64_t o_final;                                 // both
  uint32_t tmem_base;
  uint32_t n_union;
  uint32_t last_ragged;
};
static_assert(sizeof(Bars) <= 256, "barrier block");

struct UnionWalk4 {
  const uint32_t *m;
  int w;
  uint32_t rem;
  BA_DEVICE uint32_t word(int i) const { return m[i] | m[kMaskWords + i] | m[2 * kMaskWords + i] | m[3 * kMaskWords + i]; }
  BA_DEVICE void init(const uint32_t *m_) { m = m_; w = 0; rem = word(0); }
  BA_DEVICE int next() {
    while (rem == 0) { ++w; rem = word(w); }
    const int bit = __ffs(rem) - 1;
    rem &= rem - 1;
    return w * 32 + bit;
  }
};

template <int kEmu>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
attn_pp2_kernel(const AttnArgs a, const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_v) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = smem_u32(smem);
  if (base & 1023u) __trap();
  Bars &bars = *reinterpret_cast<Bars *>(smem + SMEM_BARS);
  uint32_t *mask = reinterpret_cast<uint32_t *>(smem + SMEM_MASK);  // [blk][word], blk = block - 4q

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int64_t quad = blockIdx.x >> 1;
  const int64_t bh = blockIdx.y;
  const int64_t b = bh / a.hq, h = bh - b * a.hq;
  const int64_t hk = h / (a.hq / a.hkv);
  const int nw = (int)((a.nk + 31) >> 5);
  const int64_t g0 = 4 * quad;  // first query block of the quad

  // ---- key-block sets of the four query blocks as bitmasks (both CTAs build all four)
  for (int w = threadIdx.x; w < 4 * kMaskWords; w += kThreads) mask[w] = 0u;
  __syncthreads();
  for (int q4 = 0; q4 < 4; ++q4) {
    if (g0 + q4 >= a.nq) break;
    const int64_t row = bh * a.nq + g0 + q4;
    uint32_t *m = mask + q4 * kMaskWords;
    if (a.kv_index) {
      const int cnt = a.kv_count ? a.kv_count[row] : (int)a.kv_stride;
      if (cnt < 1 && threadIdx.x == 0 && (q4 & 1) == (int)rank) flag_error(a.err_flag, kErrEmptyRow);
      const int32_t *idx = a.kv_index + row * a.kv_stride;
      for (int e = threadIdx.x; e < cnt; e += kThreads) {
        const int g = idx[e];
        if ((unsigned)g >= (unsigned)a.nk) { flag_error(a.err_flag, kErrBadIndex); continue; }
        atomicOr(&m[g >> 5], 1u << (g & 31));
      }
    } else {
      for (int w = threadIdx.x; w < nw; w += kThreads)
        m[w] = (w + 1) * 32 <= a.nk ? 0xffffffffu : ((1u << (a.nk & 31)) - 1u);
    }
  }
  __syncthreads();
  if (warp == 0) {
    UnionWalk4 u4;
    u4.m = mask;
    unsigned c = 0;
    for (int w = lane; w < nw; w += 32) c += __popc(u4.word(w));
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) {
      bars.n_union = c;
      const int64_t gl = a.nk - 1;
      const bool sel_last = (u4.word((int)(gl >> 5)) >> (gl & 31)) & 1u;
      bars.last_ragged = sel_last && (a.lk - gl * (int64_t)BN) < BN;
      mbar_init(&bars.q_full, 2);
      for (int s = 0; s < NSLOT; ++s) { mbar_init(&bars.full[s], 2); mbar_init(&bars.empty[s], 1); }
      for (int s = 0; s < 2; ++s) {
        mbar_init(&bars.s_full[s], 1);
        for (int q = 0; q < kPSplit; ++q) mbar_init(&bars.p_part[s][q], 8);
      }
      mbar_init(&bars.o_final, 1);
      fence_barrier_init();
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
    }
  }
  if (warp == kMmaWarp) {  // same warp in both CTAs: paired allocation
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&bars.tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();  // barrier inits and the TMEM allocation visible to the peer CTA
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;
  const int cnt = (int)bars.n_union;

  if (warp >= 8) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsSide));
  if (warp == kProducerWarp) {
    // ================================================================ TMA producer (both CTAs)
    if (lane == 0 && cnt > 0) {
      const uint32_t qbar0 = map_to_rank(smem_u32(&bars.q_full), 0);
      if (leader) mbar_expect_tx(&bars.q_full, 2 * 2 * QTILE);  // both CTAs' two query blocks
      for (int x = 0; x < 2; ++x) {  // blocks past the end of the sequence are zero-filled
        const int g = (int)(g0 + 2 * x + rank);
        const uint32_t dq = base + SMEM_Q + x * QTILE;
        tma_load_4d_2sm(dq, &tm_q, qbar0, 0, g * BM, (int)h, (int)b);
        tma_load_4d_2sm(dq + QBOX, &tm_q, qbar0, 64, g * BM, (int)h, (int)b);
      }
      if (!leader) mbar_arrive_remote(qbar0);
      UnionWalk4 walk;
      walk.init(mask);
      for (int u = 0; u < cnt; ++u) {
        const int gk = walk.next();
#pragma unroll
        for (int kv = 0; kv < 2; ++kv) {  // item j = 2u + kv: K_u half, then V_u half
          const int j = 2 * u + kv, s = j % NSLOT;
          mbar_wait(&bars.empty[s], ((uint32_t)(j / NSLOT) & 1u) ^ 1u);
          const uint32_t fbar0 = map_to_rank(smem_u32(&bars.full[s]), 0);
          const uint32_t dst = base + SMEM_SLOT + s * HALF;
          if (leader) mbar_expect_tx(&bars.full[s], 2 * HALF);  // both halves land on CTA 0's barrier
          if (kv == 0) {  // keys [gk*128 + 64r, +64), both 64-column boxes
            tma_load_4d_2sm(dst, &tm_k, fbar0, 0, gk * BN + 64 * (int)rank, (int)hk, (int)b);
            tma_load_4d_2sm(dst + KBOX, &tm_k, fbar0, 64, gk * BN + 64 * (int)rank, (int)hk, (int)b);
          } else {        // keys [gk*128, +128), value columns [64r, +64)
            tma_load_4d_2sm(dst, &tm_v, fbar0, 64 * (int)rank, gk * BN, (int)hk, (int)b);
          }
          if (!leader) mbar_arrive_remote(fbar0);
        }
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    // ================================================================ MMA issuer (CTA 0)
    if (leader && lane == 0 && cnt > 0) {
      mbar_wait(&bars.q_full, 0);
      tc_fence_after();
      auto slot_addr = [&](int j) { return base + SMEM_SLOT + (j % NSLOT) * HALF; };
      auto wait_full = [&](int j) {
        mbar_wait(&bars.full[j % NSLOT], (uint32_t)(j / NSLOT) & 1u);
        tc_fence_after();
      };
      auto issue_s = [&](int x, int u) {  // S_x = Q_x K_u^T, M = 256 over both SMs
        const uint64_t dq = make_desc(base + SMEM_Q + x * QTILE, 16, 1024), dk = make_desc(slot_addr(2 * u), 16, 1024);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint64_t oq = ((kk >> 2) * QBOX + (kk & 3) * 32) >> 4, ok = ((kk >> 2) * KBOX + (kk & 3) * 32) >> 4;
          mma_ss_2sm(tmem + s_col(x), dq + oq, dk + ok, IDESC_S, kk > 0 ? 1u : 0u);
        }
        mma_commit_2sm_mc(&bars.s_full[x], 0x3);
      };
      auto issue_pv = [&](int x, int u, int part) {  // O_x += P_x V_u, P_x from TMEM (each SM its rows)
        const uint64_t dv = make_desc(slot_addr(2 * u + 1), HALF, 1024);
        constexpr int KPP = BN / 16 / kPSplit;
#pragma unroll
        for (int kk = KPP * part; kk < KPP * part + KPP; ++kk)
          mma_ts_2sm(tmem + O_COL0 + 128 * x, tmem + s_col(x) + kk * 8, dv + (uint64_t)((kk * 2048) >> 4), IDESC_O,
                     (u > 0 || kk > 0) ? 1u : 0u);
      };
      wait_full(0);
      issue_s(0, 0);
      issue_s(1, 0);
      mma_commit_2sm_mc(&bars.empty[0], 0x3);  // K_0 read by both
      for (int u = 0; u < cnt; ++u) {
        const bool next = u + 1 < cnt;
        mbar_wait(&bars.p_part[0][0], (uint32_t)u & 1u);  // both CTAs' softmax 0 wrote P_0(u), first part
        wait_full(2 * u + 1);
        issue_pv(0, u, 0);
#pragma unroll
        for (int q = 1; q < kPSplit; ++q) {
          mbar_wait(&bars.p_part[0][q], (uint32_t)u & 1u);
          tc_fence_after();
          issue_pv(0, u, q);
        }
        if (next) {
          wait_full(2 * u + 2);
          issue_s(0, u + 1);  // S_0 buffer reuse: after PV_0(u) in issue order
        }
#pragma unroll
        for (int q = 0; q < kPSplit; ++q) {
          mbar_wait(&bars.p_part[1][q], (uint32_t)u & 1u);
          tc_fence_after();
          issue_pv(1, u, q);
        }
        mma_commit_2sm_mc(&bars.empty[(2 * u + 1) % NSLOT], 0x3);  // V_u: both readers issued
        if (next) {
          issue_s(1, u + 1);
          mma_commit_2sm_mc(&bars.empty[(2 * u + 2) % NSLOT], 0x3);  // K_{u+1}
        }
      }
      mma_commit_2sm_mc(&bars.o_final, 0x3);
    }
    __syncwarp();
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsSoftmax));
    // ================================================================ softmax + epilogue (both CTAs)
    const int x = warp >> 2;            // MMA / block slot of this warpgroup
    const int qd = warp & 3;            // TMEM lane quadrant
    const int r = qd * 32 + lane;       // row within the query block
    const uint32_t trow = tmem + ((uint32_t)(qd * 32) << 16);
    const uint32_t scol = s_col(x), ocol = O_COL0 + 128 * x;
    const int64_t g = g0 + 2 * x + rank;  // this warpgroup's query block
    const int64_t row0 = g * (int64_t)BM;
    const int nrows = (int)imin64(BM, a.lq - row0);  // <= 0 past the end of the sequence
    const uint32_t *my_mask = mask + (2 * x + rank) * kMaskWords;
    const bool last_ragged = bars.last_ragged != 0u;
    const int64_t ragged_valid = a.lk - (a.nk - 1) * (int64_t)BN;
    const float c = a.scale * 1.4426950408889634f;
    float m = -INFINITY, l = 0.f;
    uint32_t sr[128];
    uint32_t pbar0[kPSplit];
#pragma unroll
    for (int q = 0; q < kPSplit; ++q) pbar0[q] = map_to_rank(smem_u32(&bars.p_part[x][q]), 0);
    UnionWalk4 walk;
    walk.init(mask);
    // P (bf16 pairs) over S in TMEM: part q = keys 64q .. -> columns 32q .., then an arrive on
    // CTA 0's p_part[x][q] (the MMA is issued by CTA 0 for both SMs)
    auto publish_part = [&](int q) {
      tmem_st_x32(trow + scol + 32 * q, sr + 32 * q);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(pbar0[q]);
    };
    for (int u = 0; u < cnt; ++u) {
      const int gk = walk.next();
      const bool mine = (my_mask[gk >> 5] >> (gk & 31)) & 1u;  // warpgroup-uniform
      mbar_wait(&bars.s_full[x], (uint32_t)u & 1u);
      tc_fence_after();
      if (mine) {
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) tmem_ld_x32(trow + scol + q4 * 32, sr + q4 * 32);
        tmem_wait_ld();
        if (last_ragged && u == cnt - 1) {
#pragma unroll
          for (int i = 0; i < 128; ++i)
            if (i >= ragged_valid) sr[i] = __float_as_uint(-INFINITY);
        }
        float m8[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) m8[v] = fmaxf(__uint_as_float(sr[2 * v]), __uint_as_float(sr[2 * v + 1]));
#pragma unroll
        for (int i = 16; i < 128; i += 16) {
#pragma unroll
          for (int v = 0; v < 8; ++v) m8[v] = fmax3(m8[v], __uint_as_float(sr[i + 2 * v]), __uint_as_float(sr[i + 2 * v + 1]));
        }
        const float mt = fmax3(fmax3(m8[0], m8[1], m8[2]), fmax3(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7])) * c;
        if (m == -INFINITY) {
          m = mt;  // first tile of these rows: O rows are still zero (earlier P rows were 0)
        } else {
          const bool need = mt > m + kRescaleThreshold;
          if (__any_sync(0xffffffffu, need)) {
            // PV_x(u-1) is complete: the commit behind s_full[x](u) tracks every earlier MMA
            float corr = 1.f;
            if (need) { corr = ex2(m - mt); m = mt; }
            uint32_t ov[16];
#pragma unroll
            for (int q8 = 0; q8 < 8; ++q8) {
              tmem_ld_x16(trow + ocol + q8 * 16, ov);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 16; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * corr);
              tmem_st_x16(trow + ocol + q8 * 16, ov);
            }
            l *= corr;
          }
        }
        const uint64_t c2 = f2(c, c), nm2 = f2(-m, -m);
        uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
        for (int h2 = 0; h2 < kPSplit; ++h2) {
#pragma unroll
          for (int i = 32 * h2; i < 32 * h2 + 32; ++i) {
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
          if (h2 < kPSplit - 1) publish_part(h2);
        }
        const uint64_t t2 = fadd2(fadd2(acc2[0], acc2[1]), fadd2(acc2[2], acc2[3]));
        float a0, a1;
        unf2(t2, a0, a1);
        l += a0 + a1;
      } else {
#pragma unroll
        for (int i = 0; i < 64; ++i) sr[i] = 0u;  // block not selected by these rows: P = 0
#pragma unroll
        for (int q = 0; q < kPSplit - 1; ++q) publish_part(q);
      }
      publish_part(kPSplit - 1);
    }
    if (cnt > 0) {
      mbar_wait(&bars.o_final, 0);
      tc_fence_after();
    }
    const float inv = l > 0.f ? 1.f / l : 0.f;
    int64_t orow = row0 + r;
    if (r < nrows && a.perm_q) orow = a.perm_q[bh * a.lq + row0 + r];
    const int64_t o_off = b * a.os[0] + h * a.os[1] + orow * a.os[2];
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      uint32_t ov[32];
      tmem_ld_x32(trow + ocol + q4 * 32, ov);
      tmem_wait_ld();
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)  // l == 0 (empty row): zeros, never unwritten TMEM x 0
        pk[i] = l > 0.f ? pack_bf16(__uint_as_float(ov[2 * i]) * inv, __uint_as_float(ov[2 * i + 1]) * inv) : 0u;
      if (r < nrows) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          store_out_row16<__nv_bfloat16>(a, o_off + q4 * 32 + 8 * i, make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]));
      }
    }
    if (a.lse && r < nrows) a.lse[bh * a.lq + orow] = l > 0.f ? (m + log2f(l)) * 0.69314718055994531f : -INFINITY;
  }
  tc_fence_before();
  cluster_sync();  // CTA 0's MMAs wrote the peer's TMEM: both finish before either frees it
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int kEmu>
cudaError_t launch_emu(const AttnArgs &a, const CUtensorMap &mq, const CUtensorMap &mk, const CUtensorMap &mv,
                       cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_pp2_kernel<kEmu>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((unsigned)(2 * ((a.nq + 3) / 4)), (unsigned)(a.batch * a.hq));
  attn_pp2_kernel<kEmu><<<grid, kThreads, SMEM_BYTES, st>>>(a, mq, mk, mv);
  return cudaGetLastError();
}

}  // namespace pp2
}  // namespace sm100

bool attn_pp2_supported(const AttnArgs &a) {
  return a.dtype == 0 && a.d == 128 && a.B == 128 && a.nk <= 32 * sm100::pp2::kMaskWords && !a.gather;
}

cudaError_t launch_attn_pp2(const AttnArgs &a, cudaStream_t st) {
  using namespace sm100;
  CUtensorMap mq, mk, mv;
  if (!get_encode()) return cudaErrorNotSupported;
  if (!make_map(&mq, a.q, a.batch, a.hq, a.lq, a.d, a.qs, 128) || !make_map(&mk, a.k, a.batch, a.hkv, a.lk, a.d, a.ks, 64) ||
      !make_map(&mv, a.v, a.batch, a.hkv, a.lk, a.d, a.vs, 128))
    return cudaErrorInvalidValue;
  static int emu = -1;
  if (emu < 0) {
    const char *e = getenv("BA_EXP_EMU");
    emu = e ? atoi(e) : pp2::kDefaultEmu;
  }
  if (emu == 0) return pp2::launch_emu<0>(a, mq, mk, mv, st);
  if (emu == 2) return pp2::launch_emu<2>(a, mq, mk, mv, st);
  return pp2::launch_emu<1>(a, mq, mk, mv, st);
}

}  // namespace baatt
