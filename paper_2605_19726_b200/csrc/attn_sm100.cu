// attn_sm100.cu — K5: block-sparse attention on the 5th-generation tensor
// cores of sm_100a (tcgen05 + TMEM + TMA).
//
// Computes Alg. 1 steps 11-12: for a query block g_q of
// one (batch, head), O'_{g_q} = softmax(Q'_{g_q} K'_S^T * scale) V'_S over the
// key blocks S = {g_k : M_{g_q,g_k} = 1} only, renormalised
// over that support, then rows are written to the original positions pi_q(i)
// (P:566).  Non-causal.
//
// One CTA per 128-row query tile, templated on the key-block size kBN = B:
//   B = 128: the tile is one query block; it walks that block's index list.
//   B = 64:  the tile is a PAIR of adjacent query blocks (2p, 2p+1); it walks
//            the union of their two lists and every key tile is loaded once
//            for both; rows of a block that did not select the current key
//            block get P = 0.  (tcgen05 M = 128 at half the rows would waste
//            half the tensor pipe; the pair recovers it where lists overlap.)
// 11 warps:
//   warp 0     TMA producer: K_u and V_u of the u-th key block of the (union)
//              list into one stage of a 3-stage ring (128-byte swizzle, two
//              64-column boxes per tile): one "full" wait per tile for the
//              MMA issuer.  (warp 10 is idle.)
//   warp 1     MMA issuer (one elected thread) and TMEM owner.  S_u = Q K_u^T
//              with Q held in TMEM (TS form: smem carries only K and V), into
//              a double-buffered TMEM accumulator, then O += P_u V_u with P_u
//              read from TMEM — S_{u+1} overlaps the softmax of tile u.
//   warps 2-9  two softmax warpgroups; warpgroup h owns columns
//              [h*B/2, (h+1)*B/2) of every row (one thread per row and half),
//              two softmax warps per SMSP.  The halves swap partial row maxima
//              once per tile through smem + a 64-thread named barrier; online
//              softmax in the exp2 domain (FFMA2 / FMNMX3 / FADD2), lazy O
//              rescaling (only when the running max grows by > 2^8), P_u (bf16)
//              written back over S_u in TMEM in two parts per half, each
//              signalled at once so that the MMA issuer starts PV_u on it while
//              the rest is exponentiated; epilogue O / l -> bf16 rows at pi_q(i)
//              (or every peer buffer: the fused head-parallel gather), plus
//              optional LSE.
// The key-block list is turned into an smem bitmask once per CTA (union of
// the pair's lists for B = 64); every role enumerates its set bits in order.
// TMEM columns: S0 [0,B), S1 [B,2B), O [256,384), Q [384,448).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"
#include "kernels.h"
#include "sm100_ptx.cuh"

namespace baatt {
namespace sm100 {

constexpr int BM = 128;          // query rows per tile
constexpr int HD = 128;          // head dim
constexpr uint32_t O_COL = 256;
constexpr uint32_t Q_COL = 384;
constexpr int kSoftmaxWarp0 = 2;
constexpr int kThreads = 352;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
#ifndef BA_PP_SPEC
#define BA_PP_SPEC 1
#endif
constexpr bool kSpecMax = BA_PP_SPEC != 0;  // speculative row max (first P part against the running max)
constexpr int kDefaultEmu = 0;             // pairs per 8 on the polynomial exp2 (off: MUFU + power cap wins)
constexpr int kDefaultEmu64 = 0;           // dual-tile (B = 64) kernel: MUFU only (M: 1012-1020 TF/s vs 1002 at 1 of 8, 973 at 2 of 8; profiles/round2_b64_emu.json)
constexpr int kMaskWords = 1024;           // bitmask capacity: N_k <= 32768 key blocks

template <int kBN>
struct Cfg {
  static constexpr uint32_t BOX_BYTES = kBN * 64 * 2;      // kBN rows x 64 bf16 columns
  static constexpr uint32_t TILE_BYTES = 2 * BOX_BYTES;    // kBN x 128
  // one ring of (K, V) stages: a single "full" wait per tile in the MMA thread
  // (each blocking mbarrier wait costs the lone MMA issuer ~100 cycles that
  // the shallow tcgen05 queue cannot hide — tools/mma_bench.cu modes 8/9)
  static constexpr int NKV = 3 * (128 / kBN);
  static constexpr int HC = kBN / 2;                       // S columns per softmax half
  static constexpr bool kPair = kBN == 64;
  // instruction descriptors, kind::f16: D fp32, A/B bf16, dense, M = 128
  static constexpr uint32_t IDESC_S = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kBN >> 3) << 17) |
                                      ((uint32_t)(BM >> 4) << 24);                    // A K-major (Q), B K-major (K)
  static constexpr uint32_t IDESC_O = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(HD >> 3) << 17) |
                                      ((uint32_t)(BM >> 4) << 24) | (1u << 16);       // B MN-major (V: d contiguous)
  static constexpr uint32_t SMEM_KV = 0;                              // stage s: K at +0, V at +TILE_BYTES
  static constexpr uint32_t SMEM_RED = SMEM_KV + NKV * 2 * TILE_BYTES;  // float [2][2][128] row-max exchange
  static constexpr uint32_t SMEM_RED2 = SMEM_RED + 2 * 2 * 128 * 4;   // float [2][128] final l exchange
  static constexpr uint32_t SMEM_MASK = SMEM_RED2 + 2 * 128 * 4;      // uint32 [2][kMaskWords]
  static constexpr uint32_t SMEM_BARS = SMEM_MASK + 2 * kMaskWords * 4;
  static constexpr uint32_t SMEM_BYTES = SMEM_BARS + 512 + 1024;     // + alignment slack
  static __device__ constexpr uint32_t s_col(int buf) { return buf ? (uint32_t)kBN : 0u; }
};

template <int NKV>
struct __align__(8) BarsT {
  uint64_t q_full;
  uint64_t kv_full[NKV], kv_empty[NKV];
  uint64_t s_full[2], p_q[2][2][2];  // p_q[buf][column half][part]: that part's P is in TMEM (4 warps)
  uint64_t o_done;
  uint64_t o_final;  // single phase: every PV of the tile has completed (epilogue)
  uint32_t tmem_base;
  uint32_t n_union;
  uint32_t last_ragged;
};

// Ordered walk over the set bits of (A | B).
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

// kNoSoftmax: profiling-only variant (BA_ATTN_DEBUG=1) in which the softmax
// warps hand S straight back without touching it — it measures the MMA + TMA
// pipeline ceiling; its output is meaningless.
// kTrace: profiling-only variant (BA_ATTN_DEBUG=2): CTA (0,0) records clock64
// timestamps of the first kTraceTiles tiles for the producers, the MMA issuer
// and one softmax warp of each half, and prints them.
constexpr int kTraceTiles = 12;
// kDual (B = 64 only, kBN = 128 storage): every 128-key tile is TWO selected
// 64-key blocks of the union list (entries 2j and 2j+1), so S is a full
// 128 x 128 MMA (N = 128) instead of two half-width ones; softmax warpgroup hf
// owns the columns of block 2j+hf, and the row-level max / rescale state is
// advanced by both warpgroups whenever either block is selected by the rows.
// kGather (NEXT-2 zero-copy) bits: 1 = Q rows are read in place through pi_q by
// the softmax warps; 2 = K / V are the original tensors and the producer warp's
// 32 lanes fetch 4 rows each of every 128-key tile through pi_k (TMA tile::gather4).
template <int kBN, int kEmu, bool kNoSoftmax = false, bool kTrace = false, bool kDual = false, int kGather = 0>
__global__ void __launch_bounds__(kThreads, 1)
attn_sm100_kernel(const AttnArgs a, const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v) {
  using C = Cfg<kBN>;
  static_assert(!kDual || kBN == 128, "dual tiles use the 128-key storage");
  static_assert(!(kGather & 2) || kBN == 128, "gather tiles are 128 keys (B = 128, or dual B = 64)");
  constexpr bool kPairQ = C::kPair || kDual;     // a tile = query blocks (2p, 2p+1) of 64 rows
  constexpr int kBlk = kDual ? 64 : kBN;          // key-block size B
  using Bars = BarsT<C::NKV>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t *smem = smem_raw + (base - raw);
  Bars &bars = *reinterpret_cast<Bars *>(smem + C::SMEM_BARS);
  float *red = reinterpret_cast<float *>(smem + C::SMEM_RED);    // [2][2][128]
  float *red2 = reinterpret_cast<float *>(smem + C::SMEM_RED2);  // [2][128]
  uint32_t *mask_a = reinterpret_cast<uint32_t *>(smem + C::SMEM_MASK);
  uint32_t *mask_b = mask_a + kMaskWords;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x;  // 128-row query tile (one block for B = 128, a pair for B = 64)
  const int64_t bh = blockIdx.y;
  __shared__ long long trace[16][kTraceTiles];
  const bool tr = kTrace && blockIdx.x == 0 && blockIdx.y == 0;
  const long long t_origin = kTrace ? clock64() : 0;
#define TR(slot, j) do { if (tr && (j) < kTraceTiles) trace[slot][j] = clock64() - t_origin; } while (0)
  const int64_t b = bh / a.hq, h = bh - b * a.hq;
  const int64_t hk = h / (a.hq / a.hkv);
  const int nw = (int)((a.nk + 31) >> 5);

  // ---- key-block set of this tile as bitmasks (block A = first query block, B = second for pairs)
  const int64_t ga = kPairQ ? 2 * (int64_t)tile : tile;
  const bool has_b = kPairQ && ga + 1 < a.nq;
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
    } else {  // dense: every key block
      for (int w = threadIdx.x; w < nw; w += kThreads)
        m[w] = (w + 1) * 32 <= a.nk ? 0xffffffffu : ((1u << (a.nk & 31)) - 1u);
    }
  }
  __syncthreads();
  if (warp == 0) {  // |A u B| = number of key tiles this CTA streams
    unsigned c = 0;
    for (int w = lane; w < nw; w += 32) c += __popc(mask_a[w] | mask_b[w]);
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) {
      bars.n_union = c;
      // a ragged last key block, when selected, is always the last tile of the ascending walk
      const int64_t gl = a.nk - 1;
      const bool sel_last = ((mask_a[gl >> 5] | mask_b[gl >> 5]) >> (gl & 31)) & 1u;
      bars.last_ragged = sel_last && (a.lk - gl * (int64_t)kBlk) < kBlk;
    }
  }
  __syncthreads();
  const int n_blk = (int)bars.n_union;                 // selected key blocks (union)
  const int cnt = kDual ? (n_blk + 1) >> 1 : n_blk;     // key tiles streamed

  if (warp == 0 && lane == 0) {
    mbar_init(&bars.q_full, 8);   // one elected arrive per softmax warp
    for (int s = 0; s < C::NKV; ++s) { mbar_init(&bars.kv_full[s], 1); mbar_init(&bars.kv_empty[s], 1); }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars.s_full[s], 1);
      for (int q = 0; q < 4; ++q) mbar_init(&bars.p_q[s][q >> 1][q & 1], 4);
    }
    mbar_init(&bars.o_done, 1);
    mbar_init(&bars.o_final, 1);
    fence_barrier_init();
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&bars.tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;

  if (warp == 0 && (kGather & 2)) {
    // ================================================================ gather producer (zero-copy)
    if (cnt > 0) {
      const int64_t kb = (b * a.hkv + hk) * a.lk;  // pi_k row base == gather-map row base of (b, hk)
      UnionWalk walk;
      walk.init(mask_a, mask_b);
      for (int j = 0; j < cnt; ++j) {
        const int gk = walk.next();
        const int gk2 = kDual ? (2 * j + 1 < n_blk ? walk.next() : gk) : gk;
        // lane l: tile rows 4l..4l+3 (dual: lanes 0-15 -> block gk, 16-31 -> block gk2)
        const int g = (kDual && lane >= 16) ? gk2 : gk;
        const int r0 = kDual ? 4 * (lane & 15) : 4 * lane;
        int rr[4];  // the ragged tail repeats the last key row (its columns are masked to -inf)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t tok = imin64((int64_t)g * kBlk + r0 + i, a.lk - 1);
          rr[i] = (int)(kb + __ldg(a.perm_k + kb + tok));
        }
        const int s = j % C::NKV;
        mbar_wait(&bars.kv_empty[s], ((uint32_t)(j / C::NKV) & 1u) ^ 1u);
        if (lane == 0) { TR(0, j); mbar_expect_tx(&bars.kv_full[s], 2 * C::TILE_BYTES); }
        __syncwarp();
        const uint32_t dk = base + C::SMEM_KV + s * 2 * C::TILE_BYTES + lane * 512, dv = dk + C::TILE_BYTES;
        tma_gather4(dk, &tm_k, &bars.kv_full[s], 0, rr[0], rr[1], rr[2], rr[3]);
        tma_gather4(dk + C::BOX_BYTES, &tm_k, &bars.kv_full[s], 64, rr[0], rr[1], rr[2], rr[3]);
        tma_gather4(dv, &tm_v, &bars.kv_full[s], 0, rr[0], rr[1], rr[2], rr[3]);
        tma_gather4(dv + C::BOX_BYTES, &tm_v, &bars.kv_full[s], 64, rr[0], rr[1], rr[2], rr[3]);
      }
    }
    __syncwarp();
  } else if (warp == 0) {
    // ================================================================ TMA producer
    // K_u and V_u of the u-th selected key block into one stage of the ring
    const bool skip = kNoSoftmax && (a.dbg_flags & 3) == 3;  // profiling knob (no-softmax variant only)
    if (lane == 0 && cnt > 0) {
      UnionWalk walk;
      walk.init(mask_a, mask_b);
      for (int j = 0; j < cnt; ++j) {
        const int gk = walk.next();
        // dual: the second 64-key half; an odd tail reloads gk there (finite data, P = 0 columns)
        const int gk2 = kDual ? (2 * j + 1 < n_blk ? walk.next() : gk) : gk;
        const int s = j % C::NKV;
        const uint32_t ph = (uint32_t)(j / C::NKV) & 1u;
        mbar_wait(&bars.kv_empty[s], ph ^ 1u);
        TR(0, j);
        if (skip) {
          mbar_arrive(&bars.kv_full[s]);
          continue;
        }
        const uint32_t dk = base + C::SMEM_KV + s * 2 * C::TILE_BYTES, dv = dk + C::TILE_BYTES;
        mbar_expect_tx(&bars.kv_full[s], 2 * C::TILE_BYTES);
        if constexpr (kDual) {  // 64-row boxes: rows [0,64) <- block gk, rows [64,128) <- block gk2
          constexpr uint32_t HALF = 64 * 128;  // 64 rows x 128 B inside a 64-column box
#pragma unroll
          for (int hb = 0; hb < 2; ++hb) {
            const int g = hb ? gk2 : gk;
            tma_load_4d(dk + hb * HALF, &tm_k, &bars.kv_full[s], 0, g * 64, (int)hk, (int)b);
            tma_load_4d(dk + C::BOX_BYTES + hb * HALF, &tm_k, &bars.kv_full[s], 64, g * 64, (int)hk, (int)b);
            tma_load_4d(dv + hb * HALF, &tm_v, &bars.kv_full[s], 0, g * 64, (int)hk, (int)b);
            tma_load_4d(dv + C::BOX_BYTES + hb * HALF, &tm_v, &bars.kv_full[s], 64, g * 64, (int)hk, (int)b);
          }
        } else {
          tma_load_4d(dk, &tm_k, &bars.kv_full[s], 0, gk * kBN, (int)hk, (int)b);
          tma_load_4d(dk + C::BOX_BYTES, &tm_k, &bars.kv_full[s], 64, gk * kBN, (int)hk, (int)b);
          tma_load_4d(dv, &tm_v, &bars.kv_full[s], 0, gk * kBN, (int)hk, (int)b);
          tma_load_4d(dv + C::BOX_BYTES, &tm_v, &bars.kv_full[s], 64, gk * kBN, (int)hk, (int)b);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ================================================================ MMA issuer
    if (lane == 0 && cnt > 0) {
      mbar_wait(&bars.q_full, 0);
      tc_fence_after();
      auto issue_s = [&](int j) {
        const int s = j % C::NKV;
        mbar_wait(&bars.kv_full[s], (uint32_t)(j / C::NKV) & 1u);  // K_j and V_j landed
        TR(2, j);
        tc_fence_after();
        const uint32_t sk = base + C::SMEM_KV + s * 2 * C::TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * C::BOX_BYTES + (kk & 3) * 32;
          mma_ts(tmem + C::s_col(j & 1), tmem + Q_COL + kk * 8, make_desc(sk + off, 16, 1024), C::IDESC_S,
                 kk > 0 ? 1u : 0u);
        }
        mma_commit(&bars.s_full[j & 1]);
      };
      issue_s(0);
      for (int j = 0; j < cnt; ++j) {
        if (j + 1 < cnt) issue_s(j + 1);
        const int s = j % C::NKV;  // V_j arrived with K_j (waited in issue_s(j))
        const uint32_t sv = base + C::SMEM_KV + s * 2 * C::TILE_BYTES + C::TILE_BYTES;
        // PV_j in four key parts, each issued as soon as its softmax warps stored that P part:
        // (half 0, part 0), (half 1, part 0), (half 0, part 1), (half 1, part 1)
        constexpr int KH = kBN / 32, KQ = KH / 2;  // 16-key steps per column half / per part
#pragma unroll
        for (int pq = 0; pq < 4; ++pq) {
          const int hh = pq & 1, q = pq >> 1;
          mbar_wait(&bars.p_q[j & 1][hh][q], (uint32_t)(j >> 1) & 1u);
          if (pq == 0) TR(3, j);
          tc_fence_after();
#pragma unroll
          for (int t2 = 0; t2 < KQ; ++t2) {
            const int kk = hh * KH + q * KQ + t2;
            mma_ts(tmem + O_COL, tmem + C::s_col(j & 1) + kk * 8, make_desc(sv + kk * 2048, C::BOX_BYTES, 1024),
                   C::IDESC_O, (j > 0 || kk > 0) ? 1u : 0u);
          }
        }
        TR(4, j);
        mma_commit(&bars.kv_empty[s]);  // stage free once PV_j (the last reader of K_j / V_j) completes
        mma_commit(&bars.o_done);
      }
      mma_commit(&bars.o_final);
    }
    __syncwarp();
  } else if (warp >= kSoftmaxWarp0 && warp < kSoftmaxWarp0 + 8) {
    // ================================================================ softmax + epilogue
    constexpr int HC = C::HC;
    const int sw = warp - kSoftmaxWarp0;  // 0..7
    const int hf = sw >> 2;               // column half owned by this warpgroup
    const int qd = warp & 3;              // TMEM lane quadrant of this warp
    const int r = qd * 32 + lane;         // query row within the tile
    const uint32_t trow = tmem + ((uint32_t)(qd * 32) << 16);
    const int64_t row0 = (int64_t)tile * BM;
    const int nrows = (int)imin64(BM, a.lq - row0);
    // which query block of the tile this warp's rows belong to (pairs: rows 0-63 -> A, 64-127 -> B)
    const uint32_t *my_mask = (kPairQ && qd >= 2) ? mask_b : mask_a;
    // Q row half -> TMEM (A operand of S = Q K^T): element pairs packed per column
    {
      uint32_t qv[32];
      // zero-copy: Q'_i = Q_{pi_q(i)} read in place
      const int64_t qrow = (kGather & 1) ? (r < nrows ? (int64_t)__ldg(a.perm_q + bh * a.lq + row0 + r) : 0) : row0 + r;
      const __nv_bfloat16 *qp = static_cast<const __nv_bfloat16 *>(a.q) + b * a.qs[0] + h * a.qs[1] +
                                qrow * a.qs[2] + hf * 64;
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
    const float c = a.scale * 1.4426950408889634f;  // scale * log2(e)
    const int64_t ragged_valid = a.lk - (a.nk - 1) * (int64_t)kBlk;  // rows in the last key block
    float m = -INFINITY, l = 0.f;
    uint32_t sr[HC];
    const bool last_ragged = bars.last_ragged != 0u;
    UnionWalk walk;  // only pairs need the per-tile block (row-half membership)
    if constexpr (kPairQ) walk.init(mask_a, mask_b);
    for (int j = 0; j < cnt; ++j) {
      bool mine = true, active = true;  // mine: my columns are selected by my rows; active: any of the tile's
      bool ragged_here = last_ragged && j == cnt - 1;
      if constexpr (kDual) {
        const int g0 = walk.next();
        const int g1 = 2 * j + 1 < n_blk ? walk.next() : -1;
        const bool m0 = (my_mask[g0 >> 5] >> (g0 & 31)) & 1u;
        const bool m1 = g1 >= 0 && ((my_mask[g1 >> 5] >> (g1 & 31)) & 1u);
        mine = hf ? m1 : m0;
        active = m0 || m1;
        ragged_here = last_ragged && (hf ? g1 : g0) == (int)(a.nk - 1);
      } else if constexpr (C::kPair) {
        const int gk = walk.next();
        mine = (my_mask[gk >> 5] >> (gk & 31)) & 1u;  // warp-uniform
        active = mine;
      }
      mbar_wait(&bars.s_full[j & 1], (uint32_t)(j >> 1) & 1u);
      if (lane == 0 && qd == 0) TR(5 + 5 * hf, j);
      tc_fence_after();
      if constexpr (kNoSoftmax) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) { mbar_arrive(&bars.p_q[j & 1][hf][0]); mbar_arrive(&bars.p_q[j & 1][hf][1]); }
        continue;
      }
      if (mine) {
#pragma unroll
        for (int q2 = 0; q2 < HC / 32; ++q2) tmem_ld_x32(trow + C::s_col(j & 1) + hf * HC + q2 * 32, sr + q2 * 32);
        tmem_wait_ld();
        if (kDual ? ragged_here : (last_ragged && j == cnt - 1)) {
#pragma unroll
          for (int i = 0; i < HC; ++i)
            if ((kDual ? i : hf * HC + i) >= ragged_valid) sr[i] = __float_as_uint(-INFINITY);
        }
      }
      if (lane == 0 && qd == 0) TR(6 + 5 * hf, j);
      // p = 2^(s*c - m): FFMA2 for the argument, MUFU or polynomial exp2, FADD2 row sums
      const uint64_t c2 = f2(c, c);
      uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
      auto exp_pairs = [&](int i0, int i1, uint64_t nm2) {
#pragma unroll
        for (int i = i0; i < i1; ++i) {
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
      };
      constexpr int PP = HC / 4;  // packed pairs per P part (two parts per column half)
      // Speculative max (as in the pair kernel): once the running max exists, the first P part
      // is exponentiated against it while this half's max is reduced beside it, and the
      // exchange with the other half follows; the part is redone if the max grew past the
      // lazy-rescale threshold.  Iteration i reads S columns 4i..4i+3 and 2i, 2i+1, writes slot i.
      const bool spec = kSpecMax && (PP == 16 || PP == 32) && mine && m != -INFINITY;
      float pmax = -INFINITY;
      if (spec) {
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        const uint64_t nm2 = f2(-m, -m);
#pragma unroll
        for (int i = 0; i < PP; ++i) {
          constexpr int kCols = HC / PP;
#pragma unroll
          for (int t = 0; t < kCols; t += 2)
            m4[((i & 1) << 1) + ((t >> 1) & 1)] =
                fmax3(m4[((i & 1) << 1) + ((t >> 1) & 1)], __uint_as_float(sr[kCols * i + t]), __uint_as_float(sr[kCols * i + t + 1]));
          exp_pairs(i, i + 1, nm2);
        }
        pmax = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
      } else if (mine) {
        static_assert(HC % 16 == 0, "8 max chains");
        float m8[8];  // 8 independent FMNMX3 chains: latency, not issue, bounds the lone warp here
#pragma unroll
        for (int u = 0; u < 8; ++u) m8[u] = fmaxf(__uint_as_float(sr[2 * u]), __uint_as_float(sr[2 * u + 1]));
#pragma unroll
        for (int i = 16; i < HC; i += 16) {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            m8[u] = fmax3(m8[u], __uint_as_float(sr[i + 2 * u]), __uint_as_float(sr[i + 2 * u + 1]));
        }
        pmax = fmax3(fmax3(m8[0], m8[1], m8[2]), fmax3(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7]));
      }
      // swap partial maxima with the other half of the row (red is double-buffered by j;
      // every tile passes the barrier, selected or not, so the buffer reuse stays safe)
      red[((j & 1) * 2 + hf) * 128 + r] = pmax;
      tc_fence_before();
      named_bar_sync(1 + qd, 64);
      tc_fence_after();
      if (lane == 0 && qd == 0) TR(7 + 5 * hf, j);
      if (active) {
        const float mt = fmaxf(pmax, red[((j & 1) * 2 + (hf ^ 1)) * 128 + r]) * c;
        if (m == -INFINITY) {
          m = mt;  // first tile of these rows: O rows are still zero (earlier P rows were 0)
        } else {
          const bool need = mt > m + kRescaleThreshold;
          if (__any_sync(0xffffffffu, need)) {  // same rows -> same decision in both halves
            float corr = 1.f;
            if (need) { corr = ex2(m - mt); m = mt; }
            mbar_wait(&bars.o_done, (uint32_t)(j - 1) & 1u);
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
            if (spec) {  // redo the first part: its S columns [0, PP) were overwritten by P
              if constexpr (PP == 32) tmem_ld_x32(trow + C::s_col(j & 1) + hf * HC, sr);
              else if constexpr (PP == 16) tmem_ld_x16(trow + C::s_col(j & 1) + hf * HC, sr);
              tmem_wait_ld();
              if (kDual ? ragged_here : (last_ragged && j == cnt - 1)) {
#pragma unroll
                for (int i = 0; i < PP; ++i)
                  if ((kDual ? i : hf * HC + i) >= ragged_valid) sr[i] = __float_as_uint(-INFINITY);
              }
#pragma unroll
              for (int v = 0; v < 4; ++v) acc2[v] = 0ull;
              exp_pairs(0, PP, f2(-m, -m));
            }
          }
        }
      }
      // P part q of this column half (packed pairs [q*HC/4, (q+1)*HC/4)) over S in TMEM, then signal
      auto publish = [&](int q) {
        constexpr int W = HC / 4;  // TMEM columns per part
        if constexpr (W == 16) tmem_st_x16(trow + C::s_col(j & 1) + hf * (HC / 2) + q * W, sr + q * W);
        else tmem_st_x8(trow + C::s_col(j & 1) + hf * (HC / 2) + q * W, sr + q * W);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();  // all 32 lanes' P stores are complete before the warp's single arrive
        if (lane == 0) mbar_arrive(&bars.p_q[j & 1][hf][q]);
      };
      if (mine) {
        const uint64_t nm2 = f2(-m, -m);
        if (!spec) exp_pairs(0, PP, nm2);
        publish(0);  // the first part's P goes out while the second is exponentiated
        exp_pairs(PP, 2 * PP, nm2);
        const uint64_t t2 = fadd2(fadd2(acc2[0], acc2[1]), fadd2(acc2[2], acc2[3]));
        float a0, a1;
        unf2(t2, a0, a1);
        l += a0 + a1;
      } else {
#pragma unroll
        for (int i = 0; i < HC / 2; ++i) sr[i] = 0u;  // block not selected by these rows: P = 0
        publish(0);
      }
      if (lane == 0 && qd == 0) TR(8 + 5 * hf, j);
      publish(1);
      if (lane == 0 && qd == 0) TR(9 + 5 * hf, j);
    }
    // epilogue: l = sum of both halves; each half writes its 64 output columns
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
    const int64_t o_off = b * a.os[0] + h * a.os[1] + orow * a.os[2] + hf * 64;
#pragma unroll
    for (int q2 = 0; q2 < 2; ++q2) {
      uint32_t ov[32];
      tmem_ld_x32(trow + O_COL + hf * 64 + q2 * 32, ov);
      tmem_wait_ld();
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)  // lt == 0 (empty row): zeros, never unwritten TMEM x 0
        pk[i] = lt > 0.f ? pack_bf16(__uint_as_float(ov[2 * i]) * inv, __uint_as_float(ov[2 * i + 1]) * inv) : 0u;
      if (r < nrows) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          store_out_row16<__nv_bfloat16>(a, o_off + q2 * 32 + 8 * i, make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]));
      }
    }
    if (a.lse && hf == 0 && r < nrows) a.lse[bh * a.lq + orow] = lt > 0.f ? (m + log2f(lt)) * 0.69314718055994531f : -INFINITY;
  }
  tc_fence_before();
  __syncthreads();
  if (tr && threadIdx.x == 0) {
    const char *names[15] = {"prod_K", "prod_V", "mma_S", "mma_pwait", "mma_PV", "s0_wait", "s0_ld", "s0_bar",
                             "s0_exp", "s0_arr", "s1_wait", "s1_ld", "s1_bar", "s1_exp", "s1_arr"};
    for (int k = 0; k < 15; ++k) {
      printf("TRACE %-9s", names[k]);
      for (int j = 0; j < kTraceTiles && j < cnt; ++j) printf(" %7lld", trace[k][j]);
      printf("\n");
    }
  }
#undef TR
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 4-D map over a [b, H, L, d] bf16 tensor with element strides (s0, s1, s2), box 64 x rows.
bool make_map(CUtensorMap *m, const void *ptr, int64_t b, int64_t H, int64_t L, int64_t d, const int64_t *s,
              int rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)L, (cuuint64_t)H, (cuuint64_t)b};
  cuuint64_t strides[3] = {(cuuint64_t)s[2] * 2, (cuuint64_t)s[1] * 2, (cuuint64_t)s[0] * 2};
  // a zero / tiny stride on a singleton dim is legal for us but not for TMA: make it dense
  if (H == 1) strides[1] = strides[0] * (cuuint64_t)L;
  if (b == 1) strides[2] = strides[1] * (cuuint64_t)H;
  cuuint32_t box[4] = {64, (cuuint32_t)rows, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 2-D map for tile::gather4 over a [b, H, L, d] bf16 tensor that is dense across
// (batch, head) (stride[1] == L*stride[2], stride[0] == H*stride[1]): rows are
// (b*H + h)*L + t, box {64 columns, 1 row}, 128-byte swizzle.
bool make_gather_map(CUtensorMap *m, const void *ptr, int64_t b, int64_t H, int64_t L, int64_t d, const int64_t *s) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)(b * H * L)};
  cuuint64_t strides[1] = {(cuuint64_t)s[2] * 2};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int kBN, int kEmu, bool kNoSoftmax, bool kTrace, bool kDual = false, int kGather = 0>
cudaError_t launch_variant(const AttnArgs &a, const CUtensorMap &mk, const CUtensorMap &mv, cudaStream_t st) {
  using C = Cfg<kBN>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_sm100_kernel<kBN, kEmu, kNoSoftmax, kTrace, kDual, kGather>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int64_t tiles = (C::kPair || kDual) ? (a.nq + 1) / 2 : a.nq;
  dim3 grid((unsigned)tiles, (unsigned)(a.batch * a.hq));
  attn_sm100_kernel<kBN, kEmu, kNoSoftmax, kTrace, kDual, kGather><<<grid, kThreads, C::SMEM_BYTES, st>>>(a, mk, mv);
  return cudaGetLastError();
}

}  // namespace sm100

// B = 64 tile shape: "dual" (default, BA_ATTN_B64 unset) = two 64-key blocks per
// 128-key MMA tile; BA_ATTN_B64=pair = one 64-key block per (N = 64) tile.
bool attn_sm100_dual64() {
  static int v = -1;
  if (v < 0) {
    const char *bm = getenv("BA_ATTN_B64");
    v = (bm && !strcmp(bm, "pair")) ? 0 : 1;
  }
  return v == 1;
}

bool attn_sm100_supported(const AttnArgs &a) {
  return a.dtype == 0 && a.d == 128 && (a.B == 128 || a.B == 64) && a.nk <= 32 * sm100::kMaskWords;
}

cudaError_t launch_attn_sm100(const AttnArgs &a, cudaStream_t st) {
  using namespace sm100;
  CUtensorMap mk, mv;
  if (!get_encode()) return cudaErrorNotSupported;  // no TMA encoder: fail loudly, never fall back
  // exp2 offload fraction: compile-time variants, BA_EXP_EMU=0..2 selects one (tuning knob);
  // BA_ATTN_DEBUG=1 / 2 select the no-softmax / trace profiling variants (B = 128)
  static int emu = -1, dbg = -1, emu64 = -1;
  const int b64 = attn_sm100_dual64() ? 1 : 0;
  if (emu < 0) {
    const char *e64 = getenv("BA_EXP_EMU");
    emu64 = e64 ? atoi(e64) : kDefaultEmu64;
    if (emu64 < 0 || emu64 > 1) emu64 = kDefaultEmu64;
    const char *env = getenv("BA_EXP_EMU");
    emu = env ? atoi(env) : kDefaultEmu;
    if (emu < 0 || emu > 1) emu = kDefaultEmu;  // 2 of 8 measured slower (profiles/round2_b64_emu.json): not built
    const char *d = getenv("BA_ATTN_DEBUG");
    dbg = d ? atoi(d) : 0;
  }
  (void)dbg;
  if (a.gather) {  // zero-copy: B = 128 single-block tiles, or B = 64 dual tiles
    if (a.B == 64 && !attn_sm100_dual64()) return cudaErrorNotSupported;
    // same exp2-offload variant as the copy path, so both paths are bit-identical
    const int e = a.B == 64 ? emu64 : emu;
    if (a.gather & 2) {
      if (!make_gather_map(&mk, a.k, a.batch, a.hkv, a.lk, a.d, a.ks) || !make_gather_map(&mv, a.v, a.batch, a.hkv, a.lk, a.d, a.vs))
        return cudaErrorInvalidValue;
      if (a.B == 64) {
        if (e == 0) return launch_variant<128, 0, false, false, true, 3>(a, mk, mv, st);
        return launch_variant<128, 1, false, false, true, 3>(a, mk, mv, st);
      }
      if (e == 1) return launch_variant<128, 1, false, false, false, 3>(a, mk, mv, st);
      return launch_variant<128, 0, false, false, false, 3>(a, mk, mv, st);
    }
    if (!make_map(&mk, a.k, a.batch, a.hkv, a.lk, a.d, a.ks, a.B) || !make_map(&mv, a.v, a.batch, a.hkv, a.lk, a.d, a.vs, a.B))
      return cudaErrorInvalidValue;
    if (a.B == 64) {
      if (e == 0) return launch_variant<128, 0, false, false, true, 1>(a, mk, mv, st);
      return launch_variant<128, 1, false, false, true, 1>(a, mk, mv, st);
    }
    if (e == 1) return launch_variant<128, 1, false, false, false, 1>(a, mk, mv, st);
    return launch_variant<128, 0, false, false, false, 1>(a, mk, mv, st);
  }
  if (!make_map(&mk, a.k, a.batch, a.hkv, a.lk, a.d, a.ks, a.B) ||
      !make_map(&mv, a.v, a.batch, a.hkv, a.lk, a.d, a.vs, a.B))
    return cudaErrorInvalidValue;
  if (a.B == 64) {
    if (b64 == 0) return launch_variant<64, 0, false, false>(a, mk, mv, st);
#ifdef BA_PROFILING
    if (dbg == 1) {
      AttnArgs b2 = a;
      const char *sk = getenv("BA_ATTN_SKIPLOAD");
      b2.dbg_flags = sk ? atoi(sk) : 0;
      return launch_variant<128, 0, true, false, true>(b2, mk, mv, st);
    }
#endif
    switch (emu64) {  // exp2 offload for the dual-tile kernel (BA_EXP_EMU; default kDefaultEmu64)
      case 0: return launch_variant<128, 0, false, false, true>(a, mk, mv, st);
      default: return launch_variant<128, 1, false, false, true>(a, mk, mv, st);
    }
  }
#ifdef BA_PROFILING
  // profiling-only variants (build with -DBA_PROFILING): no softmax (=1), tile trace (=2)
  if (dbg == 1) {
    AttnArgs b2 = a;
    const char *sk = getenv("BA_ATTN_SKIPLOAD");
    b2.dbg_flags = sk ? atoi(sk) : 0;
    return launch_variant<128, 0, true, false>(b2, mk, mv, st);
  }
  if (dbg == 2) return launch_variant<128, 0, false, true>(a, mk, mv, st);
#endif
  switch (emu) {
    case 1: return launch_variant<128, 1, false, false>(a, mk, mv, st);
    default: return launch_variant<128, 0, false, false>(a, mk, mv, st);
  }
}

}  // namespace baatt
