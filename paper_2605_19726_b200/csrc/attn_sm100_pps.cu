// attn_sm100_pps.cu — K5 for B = 128: the ping-pong pair kernel with the next
// S MMA issued EARLY and P staged in shared memory (tcgen05 + TMEM + TMA).
//
// Computes Alg. 1 steps 11-12 exactly like
// attn_sm100_pp.cu: a CTA owns adjacent query blocks A = 2p, B = 2p+1 of one
// head and walks the union of their selected key blocks;
// rows of a block that did not select a union tile get P = 0; online softmax;
// rows written back to pi_q(i).  Non-causal.
//
// Why: in attn_sm100_pp.cu P overwrites S in TMEM, so S_X(u+1) can only be
// issued after PV_X(u) has consumed P_X(u): each block's loop is the serial
// chain softmax(u) -> PV(u) + S(u+1) on the tensor pipe -> softmax(u+1), and
// the tile trace shows ~3700 cycles per union tile against 2048 of MMA.  Here
// P goes to shared memory (SS-form PV) and the softmax releases its S buffer
// as soon as S is in registers, so S_X(u+1) runs on the tensor pipe WHILE
// softmax X(u) exponentiates; the chain per block shrinks to the softmax.
//
// TMEM (512 columns): S_A [0,128), S_B [128,256), O_A [256,384), O_B [384,512).
// SMEM: Q_A, Q_B (64 KB), P_A, P_B (64 KB, K-major 128-byte swizzle = the A
// operand layout), a 3-slot ring of 32 KB K/V tiles, bitmasks, barriers.
// Warps: 0-3 softmax A, 4-7 softmax B (one thread per row, 128 columns),
//        8 TMA producer, 9 MMA issuer + TMEM owner, 10-11 idle; setmaxnreg
//        moves registers from warpgroup 2 to the softmax warpgroups.
// MMA issue order per union tile u (X = A, then B):
//   [s_free X(u)] S_X(u+1)   [p_full X(u)] PV_X(u) -> p_empty X
// The lazy O rescale and the P store wait p_empty X(u-1) (PV_X(u-1) complete).
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

namespace pps {

constexpr int BM = 128, BN = 128, HD = 128;
constexpr uint32_t BOX = 128 * 64 * 2;       // 128 rows x 64 bf16 columns (16 KB)
constexpr uint32_t TILE = 2 * BOX;           // 128 x 128 bf16 (32 KB)
constexpr int NSLOT = 3;                     // K_0, V_0, K_1, V_1, ... (released after their last reader)
BA_DEVICE constexpr uint32_t s_col(int x) { return x ? 128u : 0u; }
constexpr uint32_t O_COL0 = 256;
constexpr int kProducerWarp = 8, kMmaWarp = 9;
constexpr int kThreads = 384;
constexpr int kRegsSoftmax = 208, kRegsSide = 80;  // 8*32*208 + 4*32*80 = 63488 <= 65536
constexpr float kRescaleThreshold = 8.0f;
constexpr int kMaskWords = 128;              // nk <= 4096 (L <= 512K tokens at B = 128)
constexpr int kDefaultEmu = 1;
constexpr uint32_t SMEM_Q = 0;               // Q_A, Q_B
constexpr uint32_t SMEM_P = 2 * TILE;        // P_A, P_B
constexpr uint32_t SMEM_SLOT = 4 * TILE;
constexpr uint32_t SMEM_MASK = SMEM_SLOT + NSLOT * TILE;
constexpr uint32_t SMEM_BARS = SMEM_MASK + 2 * kMaskWords * 4;
constexpr uint32_t SMEM_BYTES = SMEM_BARS + 256;
static_assert(SMEM_BYTES <= 232448, "exceeds the 227 KB opt-in shared memory");
// kind::f16, D fp32, A/B bf16, M = 128, N = 128; A K-major; B K-major (S: K) or MN-major (PV: V)
constexpr uint32_t IDESC_S = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
constexpr uint32_t IDESC_O = IDESC_S | (1u << 16);

struct __align__(8) Bars {
  uint64_t q_full;
  uint64_t full[NSLOT], empty[NSLOT];
  uint64_t s_full[2], s_free[2], p_full[2], p_empty[2];  // per query block (A, B)
  uint64_t o_final;
  uint32_t tmem_base;
  uint32_t n_union;
  uint32_t last_ragged;
};
static_assert(sizeof(Bars) <= 256, "barrier block");

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

// kEmu: of every 8 exp2 pairs, kEmu are evaluated by a polynomial on the FMA pipe.
template <int kEmu>
__global__ void __launch_bounds__(kThreads, 1)
attn_pps_kernel(const AttnArgs a, const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_v) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = smem_u32(smem);
  if (base & 1023u) __trap();
  Bars &bars = *reinterpret_cast<Bars *>(smem + SMEM_BARS);
  uint32_t *mask_a = reinterpret_cast<uint32_t *>(smem + SMEM_MASK);
  uint32_t *mask_b = mask_a + kMaskWords;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = blockIdx.x;
  const int64_t bh = blockIdx.y;
  const int64_t b = bh / a.hq, h = bh - b * a.hq;
  const int64_t hk = h / (a.hq / a.hkv);
  const int nw = (int)((a.nk + 31) >> 5);
  const int64_t ga = 2 * (int64_t)pair;
  const bool has_b = ga + 1 < a.nq;

  // ---- key-block sets of both query blocks as bitmasks
  for (int w = threadIdx.x; w < 2 * kMaskWords; w += kThreads) mask_a[w] = 0u;
  __syncthreads();
  for (int q2 = 0; q2 < (has_b ? 2 : 1); ++q2) {
    const int64_t row = bh * a.nq + ga + q2;
    uint32_t *m = q2 ? mask_b : mask_a;
    if (a.kv_index) {
      const int c = a.kv_count ? a.kv_count[row] : (int)a.kv_stride;
      const int32_t *idx = a.kv_index + row * a.kv_stride;
      for (int e = threadIdx.x; e < c; e += kThreads) {
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
      mbar_init(&bars.q_full, 1);
      for (int s = 0; s < NSLOT; ++s) { mbar_init(&bars.full[s], 1); mbar_init(&bars.empty[s], 1); }
      for (int s = 0; s < 2; ++s) {
        mbar_init(&bars.s_full[s], 1);
        mbar_init(&bars.s_free[s], 4);
        mbar_init(&bars.p_full[s], 4);
        mbar_init(&bars.p_empty[s], 1);
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
  const int cnt = (int)bars.n_union;

  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsSide));
    if (warp == kProducerWarp) {
      // ============================================================ TMA producer
      if (lane == 0 && cnt > 0) {
        mbar_expect_tx(&bars.q_full, 2 * TILE);
        for (int q2 = 0; q2 < 2; ++q2) {  // block B past the end of the sequence is zero-filled
          const uint32_t dq = base + SMEM_Q + q2 * TILE;
          tma_load_4d(dq, &tm_q, &bars.q_full, 0, (int)((ga + q2) * BM), (int)h, (int)b);
          tma_load_4d(dq + BOX, &tm_q, &bars.q_full, 64, (int)((ga + q2) * BM), (int)h, (int)b);
        }
        UnionWalk walk;
        walk.init(mask_a, mask_b);
        for (int u = 0; u < cnt; ++u) {
          const int gk = walk.next();
#pragma unroll
          for (int kv = 0; kv < 2; ++kv) {  // item j = 2u + kv: K_u then V_u
            const int j = 2 * u + kv, s = j % NSLOT;
            mbar_wait(&bars.empty[s], ((uint32_t)(j / NSLOT) & 1u) ^ 1u);
            const uint32_t dst = base + SMEM_SLOT + s * TILE;
            const CUtensorMap *map = kv ? &tm_v : &tm_k;
            mbar_expect_tx(&bars.full[s], TILE);
            tma_load_4d(dst, map, &bars.full[s], 0, gk * BN, (int)hk, (int)b);
            tma_load_4d(dst + BOX, map, &bars.full[s], 64, gk * BN, (int)hk, (int)b);
          }
        }
      }
      __syncwarp();
    } else if (warp == kMmaWarp) {
      // ============================================================ MMA issuer
      if (lane == 0 && cnt > 0) {
        mbar_wait(&bars.q_full, 0);
        auto slot_addr = [&](int j) { return base + SMEM_SLOT + (j % NSLOT) * TILE; };
        auto wait_full = [&](int j) {
          mbar_wait(&bars.full[j % NSLOT], (uint32_t)(j / NSLOT) & 1u);
          tc_fence_after();
        };
        auto issue_s = [&](int x, int u) {  // S_x = Q_x K_u^T into S_x's TMEM columns
          const uint32_t sq = base + SMEM_Q + x * TILE, sk = slot_addr(2 * u);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t off = (kk >> 2) * BOX + (kk & 3) * 32;
            mma_ss(tmem + s_col(x), make_desc(sq + off, 16, 1024), make_desc(sk + off, 16, 1024), IDESC_S, kk > 0 ? 1u : 0u);
          }
          mma_commit(&bars.s_full[x]);
        };
        auto issue_pv = [&](int x, int u) {  // O_x += P_x V_u, P_x from smem (K-major)
          const uint32_t sp = base + SMEM_P + x * TILE, sv = slot_addr(2 * u + 1);
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk) {
            const uint32_t off = (kk >> 2) * BOX + (kk & 3) * 32;
            mma_ss(tmem + O_COL0 + 128 * x, make_desc(sp + off, 16, 1024), make_desc(sv + kk * 2048, BOX, 1024), IDESC_O,
                   (u > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&bars.p_empty[x]);
        };
        wait_full(0);
        issue_s(0, 0);
        issue_s(1, 0);
        mma_commit(&bars.empty[0]);  // K_0 read by both
        for (int u = 0; u < cnt; ++u) {
          const bool next = u + 1 < cnt;
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            if (next) {
              mbar_wait(&bars.s_free[x], (uint32_t)u & 1u);  // softmax x holds S_x(u) in registers
              tc_fence_after();
              if (x == 0) wait_full(2 * u + 2);               // K_{u+1}
              issue_s(x, u + 1);
              if (x == 1) mma_commit(&bars.empty[(2 * u + 2) % NSLOT]);  // K_{u+1}: both readers issued
            }
            mbar_wait(&bars.p_full[x], (uint32_t)u & 1u);    // P_x(u) in smem (and O_x rescaled)
            tc_fence_after();
            if (x == 0) wait_full(2 * u + 1);                 // V_u
            issue_pv(x, u);
            if (x == 1) mma_commit(&bars.empty[(2 * u + 1) % NSLOT]);  // V_u: both readers issued
          }
        }
        mma_commit(&bars.o_final);
      }
      __syncwarp();
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsSoftmax));
    // ============================================================ softmax + epilogue
    const int x = warp >> 2;            // 0: block A, 1: block B
    const int qd = warp & 3;            // TMEM lane quadrant
    const int r = qd * 32 + lane;       // row within the query block
    const uint32_t trow = tmem + ((uint32_t)(qd * 32) << 16);
    const uint32_t scol = s_col(x), ocol = O_COL0 + 128 * x;
    const int64_t row0 = (ga + x) * (int64_t)BM;
    const int nrows = (int)imin64(BM, a.lq - row0);
    const uint32_t *my_mask = x ? mask_b : mask_a;
    const bool last_ragged = bars.last_ragged != 0u;
    const int64_t ragged_valid = a.lk - (a.nk - 1) * (int64_t)BN;
    const float c = a.scale * 1.4426950408889634f;
    // this thread's row of P in the K-major 128-byte-swizzled A-operand image:
    // 16-byte chunk q of box bx lives at bx*BOX + r*128 + ((q ^ (r & 7)) << 4)
    uint8_t *prow = smem + SMEM_P + x * TILE + r * 128;
    float m = -INFINITY, l = 0.f;
    uint32_t sr[128];
    UnionWalk walk;
    walk.init(mask_a, mask_b);
    for (int u = 0; u < cnt; ++u) {
      const int gk = walk.next();
      const bool mine = (my_mask[gk >> 5] >> (gk & 31)) & 1u;  // warpgroup-uniform
      mbar_wait(&bars.s_full[x], (uint32_t)u & 1u);
      tc_fence_after();
      if (mine) {
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) tmem_ld_x32(trow + scol + q4 * 32, sr + q4 * 32);
        tmem_wait_ld();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.s_free[x]);  // S_x may be overwritten by S_x(u+1)
      float corr = 1.f;
      bool rescale = false;
      if (mine) {
        if (last_ragged && u == cnt - 1) {
#pragma unroll
          for (int i = 0; i < 128; ++i)
            if (i >= ragged_valid) sr[i] = __float_as_uint(-INFINITY);
        }
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int i = 0; i < 128; i += 8) {
#pragma unroll
          for (int v = 0; v < 4; ++v) m4[v] = fmax3(m4[v], __uint_as_float(sr[i + 2 * v]), __uint_as_float(sr[i + 2 * v + 1]));
        }
        const float mt = fmaxf(fmax3(m4[0], m4[1], m4[2]), m4[3]) * c;
        if (m == -INFINITY) {
          m = mt;  // first tile of these rows: O rows are still zero (earlier P rows were 0)
        } else {
          const bool need = mt > m + kRescaleThreshold;
          rescale = __any_sync(0xffffffffu, need);
          if (need) { corr = ex2(m - mt); m = mt; }
          l *= corr;
        }
        const uint64_t c2 = f2(c, c), nm2 = f2(-m, -m);
        uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
        for (int i = 0; i < 64; ++i) {
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
        for (int i = 0; i < 64; ++i) sr[i] = 0u;  // block not selected by these rows: P = 0
      }
      // PV_x(u-1) must be complete before P_x is overwritten and before O_x is rescaled
      if (u > 0) mbar_wait(&bars.p_empty[x], (uint32_t)(u - 1) & 1u);
      tc_fence_after();
      if (rescale) {
        uint32_t ov[16];
#pragma unroll
        for (int q8 = 0; q8 < 8; ++q8) {
          tmem_ld_x16(trow + ocol + q8 * 16, ov);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * corr);
          tmem_st_x16(trow + ocol + q8 * 16, ov);
        }
        tmem_wait_st();
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) {  // 16 chunks of 8 bf16: box q >> 3, chunk q & 7
        const uint32_t off = (q >> 3) * BOX + (((q & 7) ^ (r & 7)) << 4);
        *reinterpret_cast<uint4 *>(prow + off) = make_uint4(sr[4 * q], sr[4 * q + 1], sr[4 * q + 2], sr[4 * q + 3]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy P stores -> UMMA reads
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.p_full[x]);
    }
    if (cnt > 0) {
      mbar_wait(&bars.o_final, 0);
      tc_fence_after();
    }
    const float inv = l > 0.f ? 1.f / l : 0.f;
    int64_t orow = row0 + r;
    if (r < nrows && a.perm_q) orow = a.perm_q[bh * a.lq + row0 + r];
    __nv_bfloat16 *o = static_cast<__nv_bfloat16 *>(a.out) + b * a.os[0] + h * a.os[1] + orow * a.os[2];
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      uint32_t ov[32];
      tmem_ld_x32(trow + ocol + q4 * 32, ov);
      tmem_wait_ld();
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(__uint_as_float(ov[2 * i]) * inv, __uint_as_float(ov[2 * i + 1]) * inv);
      if (r < nrows) {
        uint4 *dst = reinterpret_cast<uint4 *>(o + q4 * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
      }
    }
    if (a.lse && r < nrows) a.lse[bh * a.lq + orow] = l > 0.f ? (m + log2f(l)) * 0.69314718055994531f : -INFINITY;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int kEmu>
cudaError_t launch_emu(const AttnArgs &a, const CUtensorMap &mq, const CUtensorMap &mk, const CUtensorMap &mv, dim3 grid,
                       cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_pps_kernel<kEmu>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  attn_pps_kernel<kEmu><<<grid, kThreads, SMEM_BYTES, st>>>(a, mq, mk, mv);
  return cudaGetLastError();
}

}  // namespace pps
}  // namespace sm100

bool attn_pps_supported(const AttnArgs &a) {
  return a.dtype == 0 && a.d == 128 && a.B == 128 && !a.gather && a.nk <= 32 * sm100::pps::kMaskWords;
}

cudaError_t launch_attn_pps(const AttnArgs &a, cudaStream_t st) {
  using namespace sm100;
  using namespace sm100::pps;
  CUtensorMap mq, mk, mv;
  if (!get_encode()) return cudaErrorNotSupported;
  if (!make_map(&mq, a.q, a.batch, a.hq, a.lq, a.d, a.qs, 128) || !make_map(&mk, a.k, a.batch, a.hkv, a.lk, a.d, a.ks, 128) ||
      !make_map(&mv, a.v, a.batch, a.hkv, a.lk, a.d, a.vs, 128))
    return cudaErrorInvalidValue;
  static int emu = -1;
  if (emu < 0) {
    const char *e = getenv("BA_EXP_EMU");
    emu = e ? atoi(e) : kDefaultEmu;
    if (emu < 0 || emu > 3) emu = kDefaultEmu;
  }
  dim3 grid((unsigned)((a.nq + 1) / 2), (unsigned)(a.batch * a.hq));
  switch (emu) {
    case 0: return launch_emu<0>(a, mq, mk, mv, grid, st);
    case 2: return launch_emu<2>(a, mq, mk, mv, grid, st);
    case 3: return launch_emu<3>(a, mq, mk, mv, grid, st);
    default: return launch_emu<1>(a, mq, mk, mv, grid, st);
  }
}

}  // namespace baatt
