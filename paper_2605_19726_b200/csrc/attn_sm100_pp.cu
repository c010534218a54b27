// attn_sm100_pp.cu — K5 for B = 128: one CTA, a PAIR of query blocks,
// ping-pong between them (tcgen05 + TMEM + TMA, sm_100a).
//
// Computes Alg. 1 steps 11-12: each query block attends
// over its selected key blocks only, online softmax, rows
// written back to pi_q(i).  Non-causal.
//
// A CTA owns the adjacent query blocks A = 2p and B = 2p+1 of one head and
// walks their two index lists in lock step (PairWalk): first the key blocks
// both selected (norm-sorted neighbours select nearly the same ones: the union
// of the two lists is 1.01 kappa at A and C), each K/V tile loaded once for
// both; then the blocks only A selected paired with the blocks only B selected,
// two different tiles per step.  With equal list lengths (top-kappa) every step
// is useful work for both blocks however incoherent the lists are; only an
// unequal tail (top-p, kv_count) runs one block with P = 0.
//
// Why the pair: the lone MMA-issuing thread pays ~100 cycles per blocking
// mbarrier wait that the shallow tcgen05 queue cannot hide (tools/mma_bench.cu
// modes 6-10), and the softmax of one 128 x 128 tile is MUFU-bound at 1024
// cycles per SM.  Alternating A and B gives the tensor pipe independent work
// during each softmax (FA4-style ping-pong) and 32 MMAs per K/V wait; each
// softmax warpgroup owns whole rows (no cross-warp max exchange).
//
// Warps: 0-3 softmax of block A, 4-7 softmax of block B (one thread per row,
//        128 columns; warp w reads TMEM lane quadrant w % 4),
//        8 TMA producer (Q_A, Q_B once; then K_u, V_u into a 5-slot ring),
//        9 MMA issuer (one elected thread) + TMEM owner, 10-11 idle.
//        setmaxnreg moves registers from warpgroup 2 (warps 8-11: 80 each) to
//        the softmax warpgroups (208 each): a 128-column S row per thread and
//        the exp-offload polynomial fit without spills.
// TMEM: S_A [0,128), S_B [128,256), O_A [256,384), O_B [384,512).
// Issue order per union tile u:
//   PV_A(u-1) | S_A(u) | PV_B(u-1) | S_B(u)      (softmax A(u) || PV_B, S_B)
// The commit that signals S_X(u) tracks every earlier MMA, so PV_X(u-1) is
// complete whenever softmax X starts tile u: the lazy O rescale needs no wait.
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
bool make_gather_map(CUtensorMap *m, const void *ptr, int64_t b, int64_t H, int64_t L, int64_t d, const int64_t *s);
PFN_cuTensorMapEncodeTiled_v12000 get_encode();

namespace pp {

constexpr int BM = 128, BN = 128, HD = 128;
constexpr uint32_t BOX = 128 * 64 * 2;       // 128 rows x 64 bf16 columns (16 KB)
constexpr uint32_t TILE = 2 * BOX;           // 128 x 128 bf16 (32 KB)
// K/V ring of 32 KB slots filled in the MMA's consumption order: per step u a
// shared tile is K_u, V_u; a split step K_A(u), K_B(u), V_A(u), V_B(u).  A slot is
// released by a commit after its last reader (shared K_u after S_B(u), V_u after
// PV_B(u); split: each after its one reader), so 5 slots keep 1-2 steps in flight.
constexpr int NSLOT = 5;
BA_DEVICE constexpr uint32_t s_col(int x) { return x ? 128u : 0u; }
constexpr uint32_t O_COL0 = 256;
constexpr int kProducerWarp = 8, kMmaWarp = 9;
#ifndef BA_PP_PSPLIT
#define BA_PP_PSPLIT 2
#endif
constexpr int kPSplit = BA_PP_PSPLIT;     // P handed to the MMA in this many key parts (2: +5% over 1; 4: -2% vs 2)
constexpr int kThreads = 384;             // 12 warps: 8 softmax (warpgroups 0, 1) + warpgroup 2 (producer, MMA, 2 idle)
constexpr int kRegsSoftmax = 208, kRegsSide = 80;  // setmaxnreg: 8*32*208 + 4*32*80 = 63488 <= 65536
constexpr float kRescaleThreshold = 8.0f;
#ifndef BA_PP_EMU0
#define BA_PP_EMU0 -1
#endif
#ifndef BA_PP_EMU1
#define BA_PP_EMU1 -1
#endif
#ifndef BA_PP_DEFER_SUM
#define BA_PP_DEFER_SUM 1
#endif
constexpr bool kDeferSum = BA_PP_DEFER_SUM != 0;
#ifndef BA_PP_RELOAD
#define BA_PP_RELOAD 0
#endif
// BA_PP_RELOAD=1: S of P part 1 re-read from TMEM after part 0 is published.  Without it ptxas
// hoists most of part 1's exps above the first publish (101 of 112 MUFU.EX2 before the first
// STTM), so both parts go out nearly together; with it the SASS is in program order, but the
// attention rate is unchanged (A +0.2%, C +-0; profiles/round2_tmem_reload_ab.txt): off.
constexpr bool kReload = BA_PP_RELOAD != 0;
static_assert(!kReload || kPSplit == 2, "the reload covers keys 64..127: kPSplit 2");
static_assert(kPSplit >= 2, "the first P part is published before the remaining parts (kPSplit 1 is not a layout)");
constexpr int kMaskWords = 256;                             // nk <= 8192 (L <= 1M tokens)
constexpr int kTraceTiles = 8;
#ifndef BA_PP_TRACE_START
#define BA_PP_TRACE_START 32
#endif
constexpr int kTraceStart = BA_PP_TRACE_START;  // first traced step (past the pipeline fill)
constexpr int kDefaultEmu = 1;  // 1 of 8 exp2 pairs on the FMA pipe: +2.4% at A, +1.4% at C (EMU sweep, profiles/round1_microbench.txt)
constexpr uint32_t SMEM_Q = 0;                              // Q_A, Q_B
constexpr uint32_t SMEM_SLOT = 2 * TILE;
constexpr uint32_t SMEM_MASK = SMEM_SLOT + NSLOT * TILE;
constexpr uint32_t SMEM_BARS = SMEM_MASK + 2 * kMaskWords * 4;
constexpr uint32_t SMEM_TRACE = SMEM_BARS + 256;
constexpr uint32_t SMEM_BYTES = SMEM_TRACE + 12 * kTraceTiles * 8;
static_assert(SMEM_BYTES <= 232448, "exceeds the 227 KB opt-in shared memory");
// kind::f16, D fp32, A/B bf16, M = 128, N = 128
constexpr uint32_t IDESC_S = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
constexpr uint32_t IDESC_O = IDESC_S | (1u << 16);  // B = V MN-major (N = d = 128)

struct __align__(8) Bars {
  uint64_t q_full;
  uint64_t full[NSLOT], empty[NSLOT];
  uint64_t s_full[2], p_part[2][kPSplit];    // per query block (A, B); p_part[q]: P of key part q in TMEM
  uint64_t o_final;
  uint32_t tmem_base;
  uint32_t n_common, n_only_a, n_only_b;  // |S_A & S_B|, |S_A \ S_B|, |S_B \ S_A|
};
static_assert(sizeof(Bars) <= 256, "barrier block");

// Ascending walk over the set bits of one of S_A & S_B (kind 0), S_A \ S_B (1), S_B \ S_A (2).
struct BitWalk {
  const uint32_t *ma, *mb;
  int w, kind;
  uint32_t rem;
  BA_DEVICE uint32_t word(int i) const {
    return kind == 0 ? (ma[i] & mb[i]) : kind == 1 ? (ma[i] & ~mb[i]) : (mb[i] & ~ma[i]);
  }
  BA_DEVICE void init(const uint32_t *a_, const uint32_t *b_, int k) { ma = a_; mb = b_; kind = k; w = 0; rem = word(0); }
  BA_DEVICE int next() {
    while (rem == 0) rem = word(++w);
    const int bit = __ffs(rem) - 1;
    rem &= rem - 1;
    return w * 32 + bit;
  }
};

// One step of the pair: key block ta for block A, tb for block B.  ta == tb: one
// shared K/V tile (2 ring items); ta != tb: two tiles (4 items).  mine_x = 0: block x
// has no key block left at this step and runs the other's tile with P = 0.
struct Step {
  int ta, tb;
  bool mine_a, mine_b;
  BA_DEVICE bool split() const { return ta != tb; }
  BA_DEVICE int items() const { return ta != tb ? 4 : 2; }
};

// The step sequence every role enumerates identically: the common blocks in
// ascending order, then the i-th block only A selected with the i-th only B
// selected.  n_steps = n_common + max(n_only_a, n_only_b).
struct PairWalk {
  BitWalk c, xa, xb;
  int u, nc, na, nb;
  BA_DEVICE void init(const uint32_t *ma, const uint32_t *mb, int nc_, int na_, int nb_) {
    c.init(ma, mb, 0); xa.init(ma, mb, 1); xb.init(ma, mb, 2);
    u = 0; nc = nc_; na = na_; nb = nb_;
  }
  BA_DEVICE Step next() {
    Step s;
    if (u < nc) {
      s.ta = s.tb = c.next();
      s.mine_a = s.mine_b = true;
    } else {
      const int i = u - nc;
      s.mine_a = i < na;
      s.mine_b = i < nb;
      const int ta = s.mine_a ? xa.next() : -1, tb = s.mine_b ? xb.next() : -1;
      s.ta = s.mine_a ? ta : tb;
      s.tb = s.mine_b ? tb : ta;
    }
    ++u;
    return s;
  }
};

// kMode: 0 product; 1 profiling-only "no softmax" (P = 0, no exps: the MMA /
// barrier / TMA skeleton alone, BA_ATTN_DEBUG=1); 2 profiling-only trace (CTA
// (0,0) prints clock64 stamps of its first kTraceTiles union tiles, BA_ATTN_DEBUG=2).
// kEmu: of every 8 exp2 pairs, kEmu are evaluated by a polynomial on the FMA
// pipe instead of MUFU (BA_EXP_EMU).
// kGather (NEXT-2 zero-copy) bits: 1 = Q, 2 = K and V are the ORIGINAL tensors,
// fetched through pi_q / pi_k by the producer warp's 32 lanes (4 rows each of
// every 128-row tile) with TMA tile::gather4 on 2-D maps over the (b*H*L, d)
// row space; otherwise tile loads of the permuted copies.
template <int kMode, int kEmu, int kGather = 0>
__global__ void __launch_bounds__(kThreads, 1)
attn_pp_kernel(const AttnArgs a, const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
               const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o) {
  // The whole 227 KB is used, so no room to realign: the dynamic window must
  // start on a 1024-byte boundary (required by the 128-byte swizzle atoms).
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = smem_u32(smem);
  if (base & 1023u) __trap();
  Bars &bars = *reinterpret_cast<Bars *>(smem + SMEM_BARS);
  uint32_t *mask_a = reinterpret_cast<uint32_t *>(smem + SMEM_MASK);
  uint32_t *mask_b = mask_a + kMaskWords;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kSlots = NSLOT;
  // exp2 offload per P part (A/B knobs BA_PP_EMU0 / BA_PP_EMU1; default kEmu for both)
  constexpr int kEmu0 = BA_PP_EMU0 >= 0 ? BA_PP_EMU0 : kEmu, kEmu1 = BA_PP_EMU1 >= 0 ? BA_PP_EMU1 : kEmu;
  constexpr bool kTrace = kMode == 2;
  // profiling-only skeletons: 1 no softmax; 3 also no K/V/Q loads (full barriers arrived
  // without a transaction: MMAs on stale shared memory); 4 also no P stores to TMEM
  constexpr bool kNoSoftmax = kMode == 1 || kMode == 3 || kMode == 4;
  constexpr bool kNoLoads = kMode == 3 || kMode == 4 || kMode == 5;  // 5: full softmax, no loads (zeroed tiles)
  long long(*trace)[kTraceTiles] = reinterpret_cast<long long(*)[kTraceTiles]>(smem + SMEM_TRACE);
  const bool tr = kTrace && blockIdx.x == 0 && blockIdx.y == 0;
  const long long t_origin = kTrace ? clock64() : 0;
#define TR(slot, j) do { if (kTrace && tr && (j) >= kTraceStart && (j) < kTraceStart + kTraceTiles) trace[slot][(j) - kTraceStart] = clock64() - t_origin; } while (0)
  const int pair = blockIdx.x;
  const int64_t bh = blockIdx.y;
  const int64_t b = bh / a.hq, h = bh - b * a.hq;
  const int64_t hk = h / (a.hq / a.hkv);
  const int nw = (int)((a.nk + 31) >> 5);
  const int64_t ga = 2 * (int64_t)pair;
  const bool has_b = ga + 1 < a.nq;

  if constexpr (kMode == 5)
    for (uint32_t i = threadIdx.x; i < SMEM_MASK / 16; i += kThreads) reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0, 0, 0, 0);
  // ---- key-block sets of both query blocks as bitmasks
  for (int w = threadIdx.x; w < 2 * kMaskWords; w += kThreads) mask_a[w] = 0u;
  __syncthreads();
  for (int q2 = 0; q2 < (has_b ? 2 : 1); ++q2) {
    const int64_t row = bh * a.nq + ga + q2;
    uint32_t *m = q2 ? mask_b : mask_a;
    if (a.kv_index) {
      const int cnt = a.kv_count ? a.kv_count[row] : (int)a.kv_stride;
      if (cnt < 1 && threadIdx.x == 0) flag_error(a.err_flag, kErrEmptyRow);  // S:393; rows -> O = 0, LSE = -inf
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
    unsigned cc = 0, ca = 0, cb = 0;
    for (int w = lane; w < nw; w += 32) {
      cc += __popc(mask_a[w] & mask_b[w]);
      ca += __popc(mask_a[w] & ~mask_b[w]);
      cb += __popc(mask_b[w] & ~mask_a[w]);
    }
    cc = __reduce_add_sync(0xffffffffu, cc);
    ca = __reduce_add_sync(0xffffffffu, ca);
    cb = __reduce_add_sync(0xffffffffu, cb);
    if (lane == 0) {
      bars.n_common = cc;
      bars.n_only_a = ca;
      bars.n_only_b = cb;
      mbar_init(&bars.q_full, (kGather & 1) ? 8 : 1);  // Q through pi_q: one arrive per softmax warp
      for (int s = 0; s < NSLOT; ++s) { mbar_init(&bars.full[s], 1); mbar_init(&bars.empty[s], 1); }
      for (int s = 0; s < 2; ++s) {
        mbar_init(&bars.s_full[s], 1);
        for (int q = 0; q < kPSplit; ++q) mbar_init(&bars.p_part[s][q], 4);
      }
      mbar_init(&bars.o_final, 1);
      fence_barrier_init();
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
    }
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&bars.tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;
  const int n_common = (int)bars.n_common, n_only_a = (int)bars.n_only_a, n_only_b = (int)bars.n_only_b;
  const int cnt = n_common + imax(n_only_a, n_only_b);  // steps

  if (warp >= 8) {
  // warpgroup 2 gives registers to the softmax warpgroups (each softmax thread holds a
  // 128-column S row); setmaxnreg is warpgroup-collective, so the role branches nest here
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsSide));
  if (warp == kProducerWarp) {
    // ================================================================ TMA producer
    // tile loads of the permuted copies by lane 0, or (kGather bits) tile::gather4 of the
    // original rows through pi by all 32 lanes, lane l fetching rows 4l..4l+3 of each tile
    if (cnt > 0) {
      const int64_t qb = bh * a.lq;                    // pi_q row base == gather-map row base of (b, h)
      const int64_t kb = (b * a.hkv + hk) * a.lk;      // same for pi_k and the K / V maps
      if constexpr (kGather & 1) {
        // Q through pi_q is loaded by the softmax warps (one row per thread, below): 64
        // serial tile::gather4 here cost ~4.5k cycles before the first MMA and queued the
        // first K/V tiles behind them in the TMA unit
      } else if (kNoLoads && lane == 0) {
        mbar_arrive(&bars.q_full);
      } else if (lane == 0) {
        mbar_expect_tx(&bars.q_full, 2 * TILE);
        for (int q2 = 0; q2 < 2; ++q2) {  // block B past the end of the sequence is zero-filled
          const uint32_t dq = base + SMEM_Q + q2 * TILE;
          tma_load_4d(dq, &tm_q, &bars.q_full, 0, (int)((ga + q2) * BM), (int)h, (int)b);
          tma_load_4d(dq + BOX, &tm_q, &bars.q_full, 64, (int)((ga + q2) * BM), (int)h, (int)b);
        }
      }
      // ring items of a step in consumption order: shared K, V; split K_A, K_B, V_A, V_B
      if constexpr (kGather & 2) {
        PairWalk walk;
        walk.init(mask_a, mask_b, n_common, n_only_a, n_only_b);
        int j = 0;
        for (int u = 0; u < cnt; ++u) {
          const Step st = walk.next();
          const int nt = st.split() ? 2 : 1;
          int rr[2][4];  // the ragged tail repeats the last key row (its columns are masked to -inf)
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const int gk = t ? st.tb : st.ta;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int64_t tok = imin64((int64_t)gk * BN + 4 * lane + i, a.lk - 1);
              rr[t][i] = (t < nt) ? (int)(kb + __ldg(a.perm_k + kb + tok)) : 0;
            }
          }
          for (int kv = 0; kv < 2; ++kv) {
            for (int t = 0; t < nt; ++t, ++j) {
              const int s = j % kSlots;
              mbar_wait(&bars.empty[s], ((uint32_t)(j / kSlots) & 1u) ^ 1u);
              if (kv == 0 && t == 0 && lane == 0) TR(0, u);
              if (lane == 0) mbar_expect_tx(&bars.full[s], TILE);
              __syncwarp();
              const uint32_t dst = base + SMEM_SLOT + s * TILE + lane * 512;
              const CUtensorMap *map = kv ? &tm_v : &tm_k;
              const int *r4 = rr[t];
              tma_gather4(dst, map, &bars.full[s], 0, r4[0], r4[1], r4[2], r4[3]);
              tma_gather4(dst + BOX, map, &bars.full[s], 64, r4[0], r4[1], r4[2], r4[3]);
            }
          }
        }
      } else if (lane == 0) {
        PairWalk walk;
        walk.init(mask_a, mask_b, n_common, n_only_a, n_only_b);
        int j = 0;
        for (int u = 0; u < cnt; ++u) {
          const Step st = walk.next();
          const int nt = st.split() ? 2 : 1;
          for (int kv = 0; kv < 2; ++kv) {
            for (int t = 0; t < nt; ++t, ++j) {
              const int s = j % kSlots, gk = t ? st.tb : st.ta;
              mbar_wait(&bars.empty[s], ((uint32_t)(j / kSlots) & 1u) ^ 1u);
              if (kv == 0 && t == 0) TR(0, u);
              if (kNoLoads) { mbar_arrive(&bars.full[s]); continue; }
              const uint32_t dst = base + SMEM_SLOT + s * TILE;
              const CUtensorMap *map = kv ? &tm_v : &tm_k;
              mbar_expect_tx(&bars.full[s], TILE);
              tma_load_4d(dst, map, &bars.full[s], 0, gk * BN, (int)hk, (int)b);
              tma_load_4d(dst + BOX, map, &bars.full[s], 64, gk * BN, (int)hk, (int)b);
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    // ================================================================ MMA issuer
    if (lane == 0 && cnt > 0) {
      mbar_wait(&bars.q_full, 0);
      auto slot_addr = [&](int j) { return base + SMEM_SLOT + (j % kSlots) * TILE; };
      auto wait_full = [&](int j) {
        mbar_wait(&bars.full[j % kSlots], (uint32_t)(j / kSlots) & 1u);
        tc_fence_after();
      };
      auto issue_s = [&](int x, int jk) {  // S_x = Q_x K^T, K in ring item jk, into S_x's TMEM columns
        // descriptors built once per tile; the K-step offsets are added to the start-address
        // field (addr >> 4, 14 bits: every smem address here is < 256 KB, so no carry out)
        const uint64_t dq = make_desc(base + SMEM_Q + x * TILE, 16, 1024), dk = make_desc(slot_addr(jk), 16, 1024);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint64_t off = ((kk >> 2) * BOX + (kk & 3) * 32) >> 4;
          mma_ss(tmem + s_col(x), dq + off, dk + off, IDESC_S, kk > 0 ? 1u : 0u);
        }
        mma_commit(&bars.s_full[x]);
      };
      // O_x += P_x V, V in ring item jv, P_x read from TMEM, in kPSplit parts of keys: each part is
      // issued as soon as the softmax has stored its P, overlapping the exps of the next part
      auto issue_pv = [&](int x, int u, int jv, int h) {
        const uint64_t dv = make_desc(slot_addr(jv), BOX, 1024);
        constexpr int KPP = BN / 16 / kPSplit;  // 16-key MMA steps per part
#pragma unroll
        for (int kk = KPP * h; kk < KPP * h + KPP; ++kk)
          mma_ts(tmem + O_COL0 + 128 * x, tmem + s_col(x) + kk * 8, dv + (uint64_t)((kk * 2048) >> 4), IDESC_O,
                 (u > 0 || kk > 0) ? 1u : 0u);
      };
      // ring items of a step starting at item j: K_A, K_B, V_A, V_B
      auto k_item = [](const Step &st, int j, int x) { return j + (st.split() ? x : 0); };
      auto v_item = [](const Step &st, int j, int x) { return j + (st.split() ? 2 + x : 1); };
      PairWalk walk;
      walk.init(mask_a, mask_b, n_common, n_only_a, n_only_b);
      Step cur = walk.next();
      int jc = 0;
      wait_full(k_item(cur, jc, 0));
      issue_s(0, k_item(cur, jc, 0));
      if (cur.split()) {
        mma_commit(&bars.empty[k_item(cur, jc, 0) % kSlots]);  // K_A(0): its one reader issued
        wait_full(k_item(cur, jc, 1));
      }
      issue_s(1, k_item(cur, jc, 1));
      mma_commit(&bars.empty[k_item(cur, jc, 1) % kSlots]);  // K_0 (or K_B(0)): every reader issued
      for (int u = 0; u < cnt; ++u) {
        const bool next = u + 1 < cnt;
        const int jn = jc + cur.items();
        Step nx = cur;
        if (next) nx = walk.next();
        mbar_wait(&bars.p_part[0][0], (uint32_t)u & 1u);  // softmax A wrote P_A(u), first key part
        TR(1, u);
        wait_full(v_item(cur, jc, 0));
        issue_pv(0, u, v_item(cur, jc, 0), 0);
#pragma unroll
        for (int q = 1; q < kPSplit; ++q) {
          mbar_wait(&bars.p_part[0][q], (uint32_t)u & 1u);
          tc_fence_after();
          issue_pv(0, u, v_item(cur, jc, 0), q);
        }
        if (cur.split()) mma_commit(&bars.empty[v_item(cur, jc, 0) % kSlots]);  // V_A(u)
        if (next) {
          wait_full(k_item(nx, jn, 0));
          issue_s(0, k_item(nx, jn, 0));  // S_A buffer reuse: after PV_A(u) in issue order
          if (nx.split()) mma_commit(&bars.empty[k_item(nx, jn, 0) % kSlots]);  // K_A(u+1)
          TR(2, u + 1);
        }
        if (cur.split()) wait_full(v_item(cur, jc, 1));
#pragma unroll
        for (int q = 0; q < kPSplit; ++q) {
          mbar_wait(&bars.p_part[1][q], (uint32_t)u & 1u);  // softmax B wrote P_B(u), key part q
          if (q == 0) TR(3, u);
          tc_fence_after();
          issue_pv(1, u, v_item(cur, jc, 1), q);
        }
        mma_commit(&bars.empty[v_item(cur, jc, 1) % kSlots]);  // V_u (or V_B(u)): every reader issued
        if (next) {
          if (nx.split()) wait_full(k_item(nx, jn, 1));
          issue_s(1, k_item(nx, jn, 1));
          mma_commit(&bars.empty[k_item(nx, jn, 1) % kSlots]);  // K_{u+1} (or K_B(u+1)): every reader issued
        }
        cur = nx;
        jc = jn;
      }
      mma_commit(&bars.o_final);
    }
    __syncwarp();
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsSoftmax));
    // ================================================================ softmax + epilogue
    const int x = warp >> 2;            // 0: block A, 1: block B
    const int qd = warp & 3;            // TMEM lane quadrant
    const int r = qd * 32 + lane;       // row within the query block
    const uint32_t trow = tmem + ((uint32_t)(qd * 32) << 16);
    const uint32_t scol = s_col(x), ocol = O_COL0 + 128 * x;
    const int64_t row0 = (ga + x) * (int64_t)BM;
    const int nrows = (int)imin64(BM, a.lq - row0);
    const int64_t ragged_valid = a.lk - (a.nk - 1) * (int64_t)BN;  // < BN: the last key block is ragged
    // PairWalk order, without walking: block x has a key block at steps u < n_common + n_only_x, and
    // the ascending walks meet the largest block N_k - 1 last (of the common blocks, or of x's own)
    const int my_only = x ? n_only_b : n_only_a;
    const int n_mine = n_common + my_only;
    int ragged_step = -1;
    if (ragged_valid < BN) {
      const int gl = (int)(a.nk - 1);
      const bool in_a = (mask_a[gl >> 5] >> (gl & 31)) & 1u, in_b = (mask_b[gl >> 5] >> (gl & 31)) & 1u;
      if (in_a && in_b) ragged_step = n_common - 1;
      else if (x ? in_b : in_a) ragged_step = n_mine - 1;
    }
    if constexpr ((kGather & 1) != 0) {
      if (cnt > 0) {
        // NEXT-2 Q in place: row r of query block x is row pi_q(row0 + r) of the original Q (rows past
        // the sequence repeat its last row; they are never stored), 16 independent 16-byte loads
        // written into the 128-byte-swizzled K-major tile the S MMA reads
        const int64_t tok = imin64(row0 + r, a.lq - 1);
        const int64_t src_row = __ldg(a.perm_q + bh * a.lq + tok);
        const uint4 *src = reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(a.q) + b * a.qs[0] +
                                                           h * a.qs[1] + src_row * a.qs[2]);
        uint4 qv[16];
#pragma unroll
        for (int c16 = 0; c16 < 16; ++c16) qv[c16] = __ldg(src + c16);
#pragma unroll
        for (int c16 = 0; c16 < 16; ++c16) {
          const int bx = c16 >> 3, cc = c16 & 7;
          *reinterpret_cast<uint4 *>(smem + SMEM_Q + x * TILE + bx * BOX + r * 128 + ((cc ^ (r & 7)) << 4)) = qv[c16];
        }
        fence_proxy_async_smem();  // generic-proxy smem writes, visible to the tensor core's reads
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.q_full);
      }
    }
    const float c = a.scale * 1.4426950408889634f;
    float m = -INFINITY, l = 0.f;
    uint32_t sr[128];
    // kDeferSum: the exps overwrite S in sr (fp32) and the packed P goes to pk; the row sum
    // is reduced after the P parts are published (off the path to the PV MMA, as cuDNN's
    // sm100 kernel does); otherwise P is packed over sr[0..63] and summed inline.
    uint32_t pk[kDeferSum ? 64 : 1];
    uint32_t *pp = kDeferSum ? pk : sr;
    // P (bf16 pairs) over S in TMEM: part q = keys 128q/kPSplit .. -> columns 64q/kPSplit ..
    // (S of those columns is already in registers), then p_part[q]
    auto publish_part = [&](int q) {
      constexpr int W = 64 / kPSplit;  // TMEM columns per part
      if constexpr (kMode != 4) {
        if constexpr (W == 32) tmem_st_x32(trow + scol + W * q, pp + W * q);
        else tmem_st_x16(trow + scol + W * q, pp + W * q);
        tmem_wait_st();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.p_part[x][q]);
    };
    for (int u = 0; u < cnt; ++u) {
      const bool mine = u < n_mine;  // warpgroup-uniform
      const bool trx = kTrace && (warp == 0 || warp == 4) && lane == 0;
      mbar_wait(&bars.s_full[x], (uint32_t)u & 1u);
      if (trx) TR(4 + 4 * x, u);
      tc_fence_after();
      if (kNoSoftmax) {
#pragma unroll
        for (int i = 0; i < 64; ++i) pp[i] = 0u;
        if (mine) l = 1.f, m = 0.f;
      } else if (mine) {
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) tmem_ld_x32(trow + scol + q4 * 32, sr + q4 * 32);
        tmem_wait_ld();
        if (trx) TR(5 + 4 * x, u);
        if (u == ragged_step) {
#pragma unroll
          for (int i = 0; i < 128; ++i)
            if (i >= ragged_valid) sr[i] = __float_as_uint(-INFINITY);
        }
        const uint64_t c2 = f2(c, c);
        uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
        // exp2 of key pairs [i0, i1) against the running max m: packed bf16 P into sr[i], sums into acc2
        auto exp_pairs = [&](int i0, int i1, uint64_t nm2) {
#pragma unroll
          for (int i = i0; i < i1; ++i) {
            const uint64_t x2 = ffma2(f2(__uint_as_float(sr[2 * i]), __uint_as_float(sr[2 * i + 1])), c2, nm2);
            uint64_t p2;
            if ((i & 7) < (i < 32 ? kEmu0 : kEmu1)) {
              p2 = exp2_poly2(x2);
            } else {
              float x0, x1;
              unf2(x2, x0, x1);
              p2 = f2(ex2(x0), ex2(x1));
            }
            float p0, p1;
            unf2(p2, p0, p1);
            if constexpr (kDeferSum) {
              sr[2 * i] = __float_as_uint(p0);
              sr[2 * i + 1] = __float_as_uint(p1);
            } else {
              acc2[i & 3] = fadd2(acc2[i & 3], p2);
            }
            pp[i] = pack_bf16(p0, p1);
          }
        };
        constexpr int PP = 64 / kPSplit;  // packed pairs per P part
        {
          // row max: 8 independent FMNMX3 chains of depth 8 (the lone warp's latency, not its issue, bounds this)
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
          exp_pairs(0, PP, f2(-m, -m));
        }
        publish_part(0);
        if (trx) TR(7 + 4 * x, u);
        const uint64_t nm2 = f2(-m, -m);
        if constexpr (kReload) {
          // S of keys 64..127 again from TMEM (P part 0 went to columns 0..31; columns 64..127 are
          // intact until the next S MMA): the loads are ordered after the tcgen05.st of part 0, so
          // ptxas cannot hoist the later parts' exps above the first publish (it does otherwise:
          // 101 of 112 MUFU.EX2 before the first STTM), and PV part 0 overlaps them as intended
#pragma unroll
          for (int q4 = 2; q4 < 4; ++q4) tmem_ld_x32(trow + scol + q4 * 32, sr + q4 * 32);
          tmem_wait_ld();
          if (u == ragged_step) {
#pragma unroll
            for (int i = 64; i < 128; ++i)
              if (i >= ragged_valid) sr[i] = __float_as_uint(-INFINITY);
          }
        }
#pragma unroll
        for (int h2 = 1; h2 < kPSplit; ++h2) {  // remaining key parts in order; each part's P goes out as soon as done
          exp_pairs(PP * h2, PP * h2 + PP, nm2);
          if (h2 < kPSplit - 1) publish_part(h2);
        }
        if constexpr (kDeferSum) {
          publish_part(kPSplit - 1);
#pragma unroll
          for (int i = 0; i < 64; ++i)
            acc2[i & 3] = fadd2(acc2[i & 3], f2(__uint_as_float(sr[2 * i]), __uint_as_float(sr[2 * i + 1])));
        }
        const uint64_t t2 = fadd2(fadd2(acc2[0], acc2[1]), fadd2(acc2[2], acc2[3]));
        float a0, a1;
        unf2(t2, a0, a1);
        l += a0 + a1;
        if (trx) TR(6 + 4 * x, u);
      } else {
#pragma unroll
        for (int i = 0; i < 64; ++i) pp[i] = 0u;  // block not selected by these rows: P = 0
#pragma unroll
        for (int q = 0; q < kPSplit - 1; ++q) publish_part(q);
      }
      if (kNoSoftmax) {
#pragma unroll
        for (int q = 0; q < kPSplit - 1; ++q) publish_part(q);
      }
      if (!kDeferSum || kNoSoftmax || !mine) publish_part(kPSplit - 1);
    }
    if (cnt > 0) {
      mbar_wait(&bars.o_final, 0);
      tc_fence_after();
    }
    const float inv = l > 0.f ? 1.f / l : 0.f;
    int64_t orow = row0 + r;
    if (r < nrows && a.perm_q) orow = a.perm_q[bh * a.lq + row0 + r];
    const int64_t o_off = b * a.os[0] + h * a.os[1] + orow * a.os[2];
    // NEXT-2 un-permute by TMA: a full block is staged in this block's (now idle) K/V ring slot
    // in the 128-byte-swizzled tile layout and written to rows pi_q(i) with tile::scatter4
    const bool scat = kMode == 0 && a.scatter && nrows == BM;  // warpgroup-uniform
    const uint32_t stage = base + SMEM_SLOT + (uint32_t)x * TILE;
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      uint32_t ov[32];
      tmem_ld_x32(trow + ocol + q4 * 32, ov);
      tmem_wait_ld();
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)  // l == 0 (empty row): zeros, never unwritten TMEM x 0
        pk[i] = l > 0.f ? pack_bf16(__uint_as_float(ov[2 * i]) * inv, __uint_as_float(ov[2 * i + 1]) * inv) : 0u;
      if (scat) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {  // 16-byte chunk cc of row r in box bx (64 columns): swizzled by r & 7
          const int c = q4 * 4 + i, bx = c >> 3, cc = c & 7;
          const uint32_t dst = stage + (uint32_t)bx * BOX + (uint32_t)r * 128u + (uint32_t)((cc ^ (r & 7)) << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(pk[4 * i]), "r"(pk[4 * i + 1]),
                       "r"(pk[4 * i + 2]), "r"(pk[4 * i + 3])
                       : "memory");
        }
      } else if (r < nrows) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          store_out_row16<__nv_bfloat16>(a, o_off + q4 * 32 + 8 * i, make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]));
      }
    }
    if (scat) {
      fence_proxy_async_smem();  // the generic-proxy smem writes, visible to the TMA unit
      named_bar_sync(3 + x, 128);
      if (qd == 0) {  // one warp: lane l scatters rows 4l .. 4l+3 of both 64-column boxes
        int rr[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t tr = row0 + 4 * lane + i;
          rr[i] = (int)(bh * a.lq + (a.perm_q ? a.perm_q[bh * a.lq + tr] : tr));
        }
#pragma unroll
        for (int bx = 0; bx < 2; ++bx)
          tma_scatter4(stage + (uint32_t)bx * BOX + (uint32_t)lane * 512u, &tm_o, 64 * bx, rr[0], rr[1], rr[2], rr[3]);
        bulk_commit();
        bulk_wait_read0();  // shared memory is read before the CTA can exit
      }
    }
    if (a.lse && r < nrows) a.lse[bh * a.lq + orow] = l > 0.f ? (m + log2f(l)) * 0.69314718055994531f : -INFINITY;
  }
  tc_fence_before();
  __syncthreads();
  if (kTrace && tr && threadIdx.x == 0) {
    const char *names[12] = {"prod_kv", "mma_pwA", "mma_SA", "mma_pwB", "A_wait", "A_ld", "A_end", "A_p0",
                             "B_wait", "B_ld", "B_end", "B_p0"};
    for (int k2 = 0; k2 < 12; ++k2) {
      printf("TRACE %-8s", names[k2]);
      for (int j = 0; j < kTraceTiles && j + kTraceStart < cnt; ++j) printf(" %7lld", trace[k2][j]);
      printf("\n");
    }
  }
#undef TR
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

}  // namespace pp
}  // namespace sm100

namespace sm100 {
namespace pp {
template <int kMode, int kEmu, int kGather = 0>
cudaError_t launch_mode(const AttnArgs &a, const CUtensorMap &mq, const CUtensorMap &mk, const CUtensorMap &mv,
                        const CUtensorMap &mo, dim3 grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_pp_kernel<kMode, kEmu, kGather>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  attn_pp_kernel<kMode, kEmu, kGather><<<grid, kThreads, SMEM_BYTES, st>>>(a, mq, mk, mv, mo);
  return cudaGetLastError();
}
}  // namespace pp
}  // namespace sm100

// BA_EXP_EMU (0..3), read once
static int emu_choice() {
  static int emu = -1;
  if (emu < 0) {
    const char *e = getenv("BA_EXP_EMU");
    emu = e ? atoi(e) : sm100::pp::kDefaultEmu;
    if (emu < 0 || emu > 1) emu = sm100::pp::kDefaultEmu;  // 2-3 of 8 measured -1..-3% (round 1-2 sweeps): not built
  }
  return emu;
}

bool attn_pp_supported(const AttnArgs &a) {
  return a.dtype == 0 && a.d == 128 && a.B == 128 && a.nk <= 32 * sm100::pp::kMaskWords;
}

cudaError_t launch_attn_pp(const AttnArgs &a, cudaStream_t st) {
  using namespace sm100;
  using namespace sm100::pp;
  CUtensorMap mq, mk, mv, mo;
  if (!get_encode()) return cudaErrorNotSupported;
  const int emu = emu_choice();
  // NEXT-2 scatter4 epilogue: O dense [b, hq, lq, d] bf16, written to `out` only (no peers / multicast)
  AttnArgs a2 = a;
  a2.scatter = 0;
  static int scat_env = -1;  // BA_PP_SCATTER=0: per-thread row stores (A/B knob)
  if (scat_env < 0) scat_env = getenv("BA_PP_SCATTER") ? atoi(getenv("BA_PP_SCATTER")) : 1;
  if (scat_env && a.out && !a.out_mc && a.n_peers == 0 && a.os[2] == a.d && a.os[1] == a.lq * a.d && a.os[0] == a.hq * a.os[1] &&
      a.lq * a.batch * a.hq < (int64_t)1 << 31 && make_gather_map(&mo, a.out, a.batch, a.hq, a.lq, a.d, a.os))
    a2.scatter = 1;
  else
    mo = mq;  // unused
  dim3 grid((unsigned)((a.nq + 1) / 2), (unsigned)(a.batch * a.hq));
  if (a.gather) {  // bit 1: Q through pi_q (gather4); bit 2: K, V through pi_k (gather4)
    const bool gq = a.gather & 1, gkv = a.gather & 2;
    const bool ok = (gq ? make_gather_map(&mq, a.q, a.batch, a.hq, a.lq, a.d, a.qs) : make_map(&mq, a.q, a.batch, a.hq, a.lq, a.d, a.qs, 128)) &&
                    (gkv ? make_gather_map(&mk, a.k, a.batch, a.hkv, a.lk, a.d, a.ks) && make_gather_map(&mv, a.v, a.batch, a.hkv, a.lk, a.d, a.vs)
                         : make_map(&mk, a.k, a.batch, a.hkv, a.lk, a.d, a.ks, 128) && make_map(&mv, a.v, a.batch, a.hkv, a.lk, a.d, a.vs, 128));
    if (!ok) return cudaErrorInvalidValue;
    // the copy path's exp2-offload variant, so both paths are bit-identical
    if (gq && gkv) return emu == 0 ? launch_mode<0, 0, 3>(a2, mq, mk, mv, mo, grid, st) : launch_mode<0, 1, 3>(a2, mq, mk, mv, mo, grid, st);
    if (gkv) return emu == 0 ? launch_mode<0, 0, 2>(a2, mq, mk, mv, mo, grid, st) : launch_mode<0, 1, 2>(a2, mq, mk, mv, mo, grid, st);
    return emu == 0 ? launch_mode<0, 0, 1>(a2, mq, mk, mv, mo, grid, st) : launch_mode<0, 1, 1>(a2, mq, mk, mv, mo, grid, st);
  }
  if (!make_map(&mq, a.q, a.batch, a.hq, a.lq, a.d, a.qs, 128) || !make_map(&mk, a.k, a.batch, a.hkv, a.lk, a.d, a.ks, 128) ||
      !make_map(&mv, a.v, a.batch, a.hkv, a.lk, a.d, a.vs, 128))
    return cudaErrorInvalidValue;
#ifdef BA_PROFILING
  // profiling-only variants (build with -DBA_PROFILING): BA_ATTN_DEBUG=1 no softmax, =2 tile trace
  static int dbg = -1;
  if (dbg < 0) {
    const char *d = getenv("BA_ATTN_DEBUG");
    dbg = d ? atoi(d) : 0;
  }
  if (dbg == 1) return launch_mode<1, 0>(a2, mq, mk, mv, mo, grid, st);
  if (dbg == 2) return launch_mode<2, kDefaultEmu>(a2, mq, mk, mv, mo, grid, st);
  if (dbg == 3) return launch_mode<3, 0>(a2, mq, mk, mv, mo, grid, st);
  if (dbg == 4) return launch_mode<4, 0>(a2, mq, mk, mv, mo, grid, st);
  if (dbg == 5) return launch_mode<5, kDefaultEmu>(a2, mq, mk, mv, mo, grid, st);
#endif
  switch (emu) {  // of every 8 exp2 pairs, emu go to the FMA-pipe polynomial
    case 0: return launch_mode<0, 0>(a2, mq, mk, mv, mo, grid, st);
    default: return launch_mode<0, 1>(a2, mq, mk, mv, mo, grid, st);
  }
}

}  // namespace baatt
