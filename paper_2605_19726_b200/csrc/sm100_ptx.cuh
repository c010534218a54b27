// sm100_ptx.cuh — inline-PTX wrappers for sm_100a (mbarrier, TMA, tcgen05
// MMA / TMEM, packed fp32x2, exp2) shared by the attention kernels.
#pragma once
#include <cuda.h>
#include <stdint.h>

#include "common.cuh"

#include "kernels.h"

namespace baatt {

// Store one 16-byte vector of an output row: to `out` (the plain case); to every peer
// buffer at the same element offset (n_peers > 0: unicast NVLink stores, the fused
// head-parallel all-gather); or ONCE to the NVLS multicast address out_mc (multimem.st:
// the NVSwitch replicates the store into every device bound to the multicast object).
template <typename T>
BA_DEVICE void store_out_row16(const AttnArgs &a, int64_t elem_off, uint4 v) {
  if (a.out_mc) {
    T *p = static_cast<T *>(a.out_mc) + elem_off;
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(__uint_as_float(v.x)),
                 "f"(__uint_as_float(v.y)), "f"(__uint_as_float(v.z)), "f"(__uint_as_float(v.w))
                 : "memory");
  } else if (a.n_peers == 0) {
    *reinterpret_cast<uint4 *>(static_cast<T *>(a.out) + elem_off) = v;
  } else {
    for (int p = 0; p < a.n_peers; ++p) *reinterpret_cast<uint4 *>(static_cast<T *>(a.out_peers[p]) + elem_off) = v;
  }
}

namespace sm100 {

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
BA_DEVICE void named_bar_sync(int id, int count) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory"); }
BA_DEVICE void named_bar_arrive(int id, int count) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory"); }


BA_DEVICE void tma_prefetch(const CUtensorMap *m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
BA_DEVICE void tma_load_4d(uint32_t dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

// TMA tile::scatter4: 4 rows of 64 bf16 columns (512 contiguous bytes of a 128-byte-swizzled
// tile in shared memory, the layout gather4 loads) to rows r0..r3 at column c0 of a 2-D map.
BA_DEVICE void tma_scatter4(uint32_t src, const CUtensorMap *m, int c0, int r0, int r1, int r2, int r3) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(src)
               : "memory");
}
BA_DEVICE void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
BA_DEVICE void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
BA_DEVICE void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// TMA tile::gather4: rows r0..r3 (row coordinate of a 2-D map), 64 columns from
// column c0 (the map's box is {64, 1}); the four rows land at dst + 128*i, with
// the map's 128-byte swizzle applied by smem address like a tile load.
BA_DEVICE void tma_gather4(uint32_t dst, const CUtensorMap *m, uint64_t *bar, int c0, int r0, int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
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
BA_DEVICE float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// Packed fp32x2 ops (FFMA2 / FADD2 on sm_100): half the issue slots of scalar fp32.
BA_DEVICE uint64_t f2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
BA_DEVICE void unf2(uint64_t v, float &lo, float &hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
BA_DEVICE uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
BA_DEVICE uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// 2^x for a pair on the FMA/ALU pipes (offloads the MUFU, FA4-style):
// x = xi + f with xi = rint(x) via the 1.5*2^23 trick, 2^f by a degree-3
// minimax polynomial on [-1/2, 1/2] (max rel. error 2.3e-4, below bf16's
// 2^-9), 2^xi added into the exponent bits.  Inputs are clamped to >= -126.
BA_DEVICE uint64_t exp2_poly2(uint64_t x2) {
  float x0, x1;
  unf2(x2, x0, x1);
  x2 = f2(fmaxf(x0, -126.f), fmaxf(x1, -126.f));
  const uint64_t magic = f2(12582912.f, 12582912.f);
  const uint64_t t = fadd2(x2, magic);
  const uint64_t xi = fadd2(t, f2(-12582912.f, -12582912.f));
  const uint64_t fr = ffma2(xi, f2(-1.f, -1.f), x2);
  uint64_t p = ffma2(f2(0.0554986224f, 0.0554986224f), fr, f2(0.243548840f, 0.243548840f));
  p = ffma2(p, fr, f2(0.693232119f, 0.693232119f));
  p = ffma2(p, fr, f2(0.999772966f, 0.999772966f));
  float p0, p1, t0, t1;
  unf2(p, p0, p1);
  unf2(t, t0, t1);
  const float r0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
  const float r1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
  return f2(r0, r1);
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



// ---- cluster helpers (2-CTA pair)
BA_DEVICE uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same smem offset in CTA `rank` of the cluster
BA_DEVICE uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// arrive on a barrier of another CTA of the cluster (plain form: a cluster-scope
// release here costs ~1000 cycles per arrive; the data it guards is TMEM,
// ordered by tcgen05.wait::st + tcgen05.fence::before_thread_sync)
BA_DEVICE void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
BA_DEVICE void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 2-SM TMA: lands in the issuing CTA's smem, completes bytes on the barrier at
// `mbar_cluster` (the leader CTA's copy of the stage barrier).
BA_DEVICE void tma_load_4d_2sm(uint32_t dst, const CUtensorMap *m, uint32_t mbar_cluster, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(mbar_cluster)
      : "memory");
}
BA_DEVICE void mma_ts_2sm(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc));
}
BA_DEVICE void mma_ss_2sm(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc));
}
// commit the issuing thread's prior tcgen05 ops to the same-offset barrier of every CTA in `mask`
BA_DEVICE void mma_commit_2sm_mc(uint64_t *bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "h"(mask)
               : "memory");
}

}  // namespace sm100
}  // namespace baatt
