// attn_sm100.cu — K5: block-sparse attention on the 5th-generation tensor
// cores of sm_100a (tcgen05 + TMEM + TMA).
//
// Computes Alg. 1 steps 11-12: for the query block g_q
// of one (batch, head), O'_{g_q} = softmax(Q'_{g_q} K'_S^T * scale) V'_S over
// the key blocks S = {g_k : M_{g_q,g_k} = 1} only,
// renormalised over that support, then rows are written to the original
// positions pi_q(i).  Non-causal.
//
// One CTA per query block (B = 128 rows, d = 128), 6 warps:
//   warp 0  TMA producer: Q once, then K_j / V_j of the j-th selected block
//           (index list kv_index) into a 2-stage ring each (128B swizzle).
//   warp 1  MMA issuer (one thread): S_j = Q K_j^T into a double-buffered
//           TMEM accumulator (SS form), then O += P_j V_j with P_j read from
//           TMEM (TS form) — so the next S overlaps this tile's softmax.
//   warps 2-5  softmax: one thread per query row; S_j TMEM -> registers,
//           online softmax in the exp2 domain with lazy O rescaling (only
//           when the running max grows by > 8, i.e. 2^8), P_j (bf16) written
//           back into the S_j columns of TMEM; epilogue O / l -> bf16 rows at
//           pi_q(i), plus optional LSE.
// TMEM: S0 cols [0,128), S1 cols [128,256), O cols [256,384) (512 allocated).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <stdio.h>

#include "common.cuh"
#include "kernels.h"

namespace baatt {
namespace sm100 {

constexpr int BM = 128;          // query rows per tile (= block size B)
constexpr int BN = 128;          // key rows per tile
constexpr int HD = 128;          // head dim
constexpr int NKS = 2;           // K stages
constexpr int NVS = 2;           // V stages
constexpr uint32_t BOX_BYTES = 128 * 64 * 2;     // one 128-row x 64-col bf16 box (16 KB)
constexpr uint32_t TILE_BYTES = 2 * BOX_BYTES;   // 128 x 128 bf16 (32 KB)
BA_DEVICE constexpr uint32_t s_col(int buf) { return buf ? 128u : 0u; }
constexpr uint32_t O_COL = 256;
constexpr int kThreads = 192;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

struct __align__(8) Bars {
  uint64_t q_full;
  uint64_t k_full[NKS], k_empty[NKS];
  uint64_t v_full[NVS], v_empty[NVS];
  uint64_t s_full[2], p_full[2];
  uint64_t o_done;
  uint32_t tmem_base;
};

constexpr uint32_t SMEM_Q = 0;
constexpr uint32_t SMEM_K = TILE_BYTES;
constexpr uint32_t SMEM_V = SMEM_K + NKS * TILE_BYTES;
constexpr uint32_t SMEM_BARS = SMEM_V + NVS * TILE_BYTES;
constexpr uint32_t SMEM_BYTES = SMEM_BARS + 256 + 1024;  // + alignment slack

// ------------------------------------------------------------------ PTX wrappers
BA_DEVICE uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

BA_DEVICE void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
BA_DEVICE void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
BA_DEVICE void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
BA_DEVICE void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
BA_DEVICE void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
BA_DEVICE void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
BA_DEVICE void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
BA_DEVICE void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
BA_DEVICE void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

BA_DEVICE void tma_prefetch(const CUtensorMap *m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
BA_DEVICE void tma_load_4d(uint32_t dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

BA_DEVICE void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc));
}
BA_DEVICE void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc));
}
BA_DEVICE void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

#include "tmem_ldst.inc"

BA_DEVICE float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
BA_DEVICE uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// UMMA shared-memory descriptor (sm_100, version 1), 128-byte swizzle.
// K-major tiles: SBO = 1024 B between 8-row groups, LBO unused (1).
// MN-major tiles: LBO = byte distance between 64-element swizzle atoms along
// MN, SBO = 1024 B between 8-row groups along K.
BA_DEVICE uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;                // version (sm_100)
  d |= 2ull << 61;                // SWIZZLE_128B
  return d;
}

// Instruction descriptor, kind::f16: D fp32, A/B bf16, dense, M = 128, N = 128.
constexpr uint32_t IDESC_BASE = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
constexpr uint32_t IDESC_S = IDESC_BASE;              // A K-major (Q), B K-major (K)
constexpr uint32_t IDESC_O = IDESC_BASE | (1u << 16); // B MN-major (V: d contiguous)

__global__ void __launch_bounds__(kThreads, 1)
attn_sm100_kernel(const AttnArgs a, const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t *smem = smem_raw + (base - raw);
  Bars &bars = *reinterpret_cast<Bars *>(smem + SMEM_BARS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = blockIdx.x;
  const int64_t bh = blockIdx.y;
  const int64_t b = bh / a.hq, h = bh - b * a.hq;
  const int64_t hk = h / (a.hq / a.hkv);
  const int64_t row = bh * a.nq + gq;
  const int cnt = a.kv_index ? (a.kv_count ? a.kv_count[row] : (int)a.kv_stride) : (int)a.nk;
  const int32_t *idx = a.kv_index ? a.kv_index + row * a.kv_stride : nullptr;

  if (warp == 0 && lane == 0) {
    mbar_init(&bars.q_full, 1);
    for (int s = 0; s < NKS; ++s) { mbar_init(&bars.k_full[s], 1); mbar_init(&bars.k_empty[s], 1); }
    for (int s = 0; s < NVS; ++s) { mbar_init(&bars.v_full[s], 1); mbar_init(&bars.v_empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&bars.s_full[s], 1); mbar_init(&bars.p_full[s], 128); }
    mbar_init(&bars.o_done, 1);
    fence_barrier_init();
    tma_prefetch(&tm_q);
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

  if (warp == 0) {
    // ================================================================ TMA producer
    if (lane == 0 && cnt > 0) {
      const uint32_t sq = base + SMEM_Q;
      mbar_expect_tx(&bars.q_full, TILE_BYTES);
      tma_load_4d(sq, &tm_q, &bars.q_full, 0, gq * BM, (int)h, (int)b);
      tma_load_4d(sq + BOX_BYTES, &tm_q, &bars.q_full, 64, gq * BM, (int)h, (int)b);
      for (int j = 0; j <= cnt; ++j) {
        if (j < cnt) {
          const int s = j % NKS;
          const uint32_t ph = (uint32_t)(j / NKS) & 1u;
          mbar_wait(&bars.k_empty[s], ph ^ 1u);
          const int gk = idx ? idx[j] : j;
          const uint32_t dst = base + SMEM_K + s * TILE_BYTES;
          mbar_expect_tx(&bars.k_full[s], TILE_BYTES);
          tma_load_4d(dst, &tm_k, &bars.k_full[s], 0, gk * BN, (int)hk, (int)b);
          tma_load_4d(dst + BOX_BYTES, &tm_k, &bars.k_full[s], 64, gk * BN, (int)hk, (int)b);
        }
        if (j >= 1) {
          const int jv = j - 1;
          const int s = jv % NVS;
          const uint32_t ph = (uint32_t)(jv / NVS) & 1u;
          mbar_wait(&bars.v_empty[s], ph ^ 1u);
          const int gk = idx ? idx[jv] : jv;
          const uint32_t dst = base + SMEM_V + s * TILE_BYTES;
          mbar_expect_tx(&bars.v_full[s], TILE_BYTES);
          tma_load_4d(dst, &tm_v, &bars.v_full[s], 0, gk * BN, (int)hk, (int)b);
          tma_load_4d(dst + BOX_BYTES, &tm_v, &bars.v_full[s], 64, gk * BN, (int)hk, (int)b);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ================================================================ MMA issuer
    if (lane == 0 && cnt > 0) {
      const uint32_t sq = base + SMEM_Q;
      mbar_wait(&bars.q_full, 0);
      auto issue_s = [&](int j) {
        const int s = j % NKS;
        mbar_wait(&bars.k_full[s], (uint32_t)(j / NKS) & 1u);
        tc_fence_after();
        const uint32_t sk = base + SMEM_K + s * TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * BOX_BYTES + (kk & 3) * 32;
          mma_ss(tmem + s_col(j & 1), make_desc(sq + off, 16, 1024), make_desc(sk + off, 16, 1024), IDESC_S,
                 kk > 0 ? 1u : 0u);
        }
        mma_commit(&bars.k_empty[s]);
        mma_commit(&bars.s_full[j & 1]);
      };
      issue_s(0);
      for (int j = 0; j < cnt; ++j) {
        if (j + 1 < cnt) issue_s(j + 1);
        mbar_wait(&bars.p_full[j & 1], (uint32_t)(j >> 1) & 1u);
        const int s = j % NVS;
        mbar_wait(&bars.v_full[s], (uint32_t)(j / NVS) & 1u);
        tc_fence_after();
        const uint32_t sv = base + SMEM_V + s * TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
          mma_ts(tmem + O_COL, tmem + s_col(j & 1) + kk * 8, make_desc(sv + kk * 2048, BOX_BYTES, 1024), IDESC_O,
                 (j > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&bars.v_empty[s]);
        mma_commit(&bars.o_done);
      }
    }
    __syncwarp();
  } else {
    // ================================================================ softmax + epilogue
    const int qd = warp & 3;             // TMEM lane quadrant of this warp
    const int r = qd * 32 + lane;        // query row within the tile
    const uint32_t trow = tmem + ((uint32_t)(qd * 32) << 16);
    const float c = a.scale * 1.4426950408889634f;  // scale * log2(e)
    const int64_t ragged_valid = a.lk - (a.nk - 1) * (int64_t)BN;  // rows in the last key block
    float m = -INFINITY, l = 0.f;
    uint32_t sr[128];
    for (int j = 0; j < cnt; ++j) {
      mbar_wait(&bars.s_full[j & 1], (uint32_t)(j >> 1) & 1u);
      tc_fence_after();
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) tmem_ld_x32(trow + s_col(j & 1) + q4 * 32, sr + q4 * 32);
      tmem_wait_ld();
      const int gk = idx ? idx[j] : j;
      if (gk == a.nk - 1 && ragged_valid < BN) {
#pragma unroll
        for (int i = 0; i < 128; ++i)
          if (i >= ragged_valid) sr[i] = __float_as_uint(-INFINITY);
      }
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < 128; ++i) mx = fmaxf(mx, __uint_as_float(sr[i]));
      const float mt = mx * c;
      float corr = 1.f;
      if (j == 0) {
        m = mt;
      } else {
        const bool need = mt > m + kRescaleThreshold;
        if (__any_sync(0xffffffffu, need)) {
          if (need) { corr = ex2(m - mt); m = mt; }
          mbar_wait(&bars.o_done, (uint32_t)(j - 1) & 1u);
          tc_fence_after();
          uint32_t ov[32];
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            tmem_ld_x32(trow + O_COL + q4 * 32, ov);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * corr);
            tmem_st_x32(trow + O_COL + q4 * 32, ov);
          }
          l *= corr;
        }
      }
      float sum = 0.f;
      const float negm = -m;
#pragma unroll
      for (int i = 0; i < 128; i += 2) {
        const float p0 = ex2(fmaf(__uint_as_float(sr[i]), c, negm));
        const float p1 = ex2(fmaf(__uint_as_float(sr[i + 1]), c, negm));
        sum += p0 + p1;
        sr[i >> 1] = pack_bf16(p0, p1);
      }
      l += sum;
      tmem_st_x32(trow + s_col(j & 1), sr);
      tmem_st_x32(trow + s_col(j & 1) + 32, sr + 32);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&bars.p_full[j & 1]);
    }
    // epilogue
    const int64_t row0 = (int64_t)gq * BM;
    const int nrows = (int)imin64(BM, a.lq - row0);
    if (cnt > 0) {
      mbar_wait(&bars.o_done, (uint32_t)(cnt - 1) & 1u);
      tc_fence_after();
    }
    const float inv = cnt > 0 ? 1.f / l : 0.f;
    int64_t orow = row0 + r;
    if (r < nrows && a.perm_q) orow = a.perm_q[bh * a.lq + row0 + r];
    __nv_bfloat16 *o = static_cast<__nv_bfloat16 *>(a.out) + b * a.os[0] + h * a.os[1] + orow * a.os[2];
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      uint32_t ov[32];
      tmem_ld_x32(trow + O_COL + q4 * 32, ov);
      tmem_wait_ld();
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)
        pk[i] = pack_bf16(__uint_as_float(ov[2 * i]) * inv, __uint_as_float(ov[2 * i + 1]) * inv);
      if (r < nrows) {
        uint4 *dst = reinterpret_cast<uint4 *>(o + q4 * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
      }
    }
    if (a.lse && r < nrows) a.lse[bh * a.lq + orow] = cnt > 0 ? (m + log2f(l)) * 0.69314718055994531f : -INFINITY;
  }
  tc_fence_before();
  __syncthreads();
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

// 4-D map over a [b, H, L, d] bf16 tensor with element strides (s0, s1, s2), box 64 x 128.
bool make_map(CUtensorMap *m, const void *ptr, int64_t b, int64_t H, int64_t L, int64_t d, const int64_t *s) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)L, (cuuint64_t)H, (cuuint64_t)b};
  cuuint64_t strides[3] = {(cuuint64_t)s[2] * 2, (cuuint64_t)s[1] * 2, (cuuint64_t)s[0] * 2};
  // a zero / tiny stride on a singleton dim is legal for us but not for TMA: make it dense
  if (H == 1) strides[1] = strides[0] * (cuuint64_t)L;
  if (b == 1) strides[2] = strides[1] * (cuuint64_t)H;
  cuuint32_t box[4] = {64, 128, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace sm100

bool attn_sm100_supported(const AttnArgs &a) { return a.dtype == 0 && a.d == 128 && a.B == 128; }

cudaError_t launch_attn_sm100(const AttnArgs &a, cudaStream_t st) {
  using namespace sm100;
  CUtensorMap mq, mk, mv;
  if (!get_encode()) return cudaErrorNotSupported;  // no TMA encoder: fail loudly, never fall back
  if (!make_map(&mq, a.q, a.batch, a.hq, a.lq, a.d, a.qs) || !make_map(&mk, a.k, a.batch, a.hkv, a.lk, a.d, a.ks) ||
      !make_map(&mv, a.v, a.batch, a.hkv, a.lk, a.d, a.vs))
    return cudaErrorInvalidValue;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(attn_sm100_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  dim3 grid((unsigned)a.nq, (unsigned)(a.batch * a.hq));
  attn_sm100_kernel<<<grid, kThreads, SMEM_BYTES, st>>>(a, mq, mk, mv);
  return cudaGetLastError();
}

}  // namespace baatt
