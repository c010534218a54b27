// select_kernels.cu — BA-Att pattern selection on sm_100a (Alg. 1 steps 1-10,
// PAPER.md P:535-562).
//
//   K1 norm_keys     key = ||x||^2 in fp32 per Q / K row (reading A4):
//                    HBM-bound, one half-warp per row, 128-bit loads, fp32
//                    partial sums (rounded mul, rounded add) combined by an
//                    xor-shuffle tree.
//   K2 radix sort    stable ascending argsort of the keys per (batch, head,
//                    window) segment (ties -> lower index):
//                    LSD radix, 4 x 8-bit passes, each = tile histogram +
//                    per-segment scan + stable tile scatter staged in smem.
//   K3 gather_stats  Q' = Q[pi_q], K' = K[pi_k], V' = V[pi_k]
//                    plus per-block mean and population variance (P:282,
//                    P:516) in fp64 from the same registers:
//                    HBM-bound, one CTA per block, coalesced 128-bit rows.
//   K4a scores       l' = Qbar.Kbar/sqrt(d) + (beta/d) sum_t (VarQ Kbar^2 +
//                    VarK Qbar^2 + VarQ VarK) (Eq. block-logit P:286-287,
//                    Eq. diag-variance-form) as ONE
//                    inner product of length 3d between the features
//                    Xq = [Qbar/sqrt(d), (beta/d)VarQ, (beta/d)Qbar^2] and
//                    Xk = [Kbar, Kbar^2 + VarK, VarK]: an fp64 SIMT micro-GEMM
//                    (64x64 tiles, 4x4 per thread) — fp64 so that masks match
//                    the fp64 oracle.
//   K4b topk         per row: max, optional m' = softmax(l'),
//                    exact kappa-th largest l' by a 64-step radix select on
//                    order-preserving bits, ties -> lower g_k, ascending index
//                    list + mask.  One warp per row, row in smem.
//                    TOPP (reading A23): kappa_row from the cumulative mass
//                    of the (-m', g_k)-ordered row, capped at kappa.
#include <math.h>
#include <stdlib.h>

#include <algorithm>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace baatt {

// =====================================================================================
// K1: norm keys.  One half-warp (16 lanes) per row; lane l owns features
// [l*d/16, (l+1)*d/16) and sums their squares sequentially in fp32; the 16
// partial sums are combined with xor offsets 8, 4, 2, 1 (a+b == b+a exactly,
// so every lane of a pair holds the oracle's p[l] + p[l+8], ...).  (An fp64
// sum cost one fp32 -> fp64 conversion per element on the XU pipe: 65% busy,
// 3.7 TB/s; the fp32 key keeps the kernel on the HBM roofline.)
// =====================================================================================
constexpr int kNormRows = 4;  // rows per half-warp: 4 independent 16-byte loads in flight per lane

template <typename T, int D>
__global__ void __launch_bounds__(256) norm_keys_kernel(const T *__restrict__ x, int64_t s0, int64_t s1,
                                                        int64_t s2, int64_t heads, int64_t L,
                                                        float *__restrict__ keys,
                                                        float *__restrict__ keys_user) {
  constexpr int PER_LANE = D / 16;  // 4 or 8 elements
  constexpr int BYTES = PER_LANE * (int)sizeof(T);
  const int lane16 = threadIdx.x & 15;
  const int64_t hw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 4;  // half-warp id
  const int64_t bh_rows = heads * L;
  const int64_t b = blockIdx.y;
  uint4 raw[kNormRows][BYTES > 16 ? 2 : 1];
  int64_t rows[kNormRows];
#pragma unroll
  for (int k = 0; k < kNormRows; ++k) {  // issue every load first
    const int64_t row = hw * kNormRows + k;
    rows[k] = row;
    if (row < bh_rows) {
      const int64_t h = row / L, t = row - h * L;
      const T *p = x + b * s0 + h * s1 + t * s2 + lane16 * PER_LANE;
      if constexpr (BYTES == 8) {
        const uint2 u = __ldg(reinterpret_cast<const uint2 *>(p));
        raw[k][0] = make_uint4(u.x, u.y, 0, 0);
      } else {
        raw[k][0] = ldg16(p);
        if constexpr (BYTES > 16) raw[k][BYTES > 16 ? 1 : 0] = ldg16(p + 16 / sizeof(T));
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kNormRows; ++k) {
    float f[PER_LANE];
    if constexpr (sizeof(T) == 2) {
      const uint32_t w[4] = {raw[k][0].x, raw[k][0].y, raw[k][0].z, raw[k][0].w};
#pragma unroll
      for (int i = 0; i < PER_LANE / 2; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
      }
    } else {
#pragma unroll
      for (int i = 0; i < PER_LANE; ++i) {
        const uint4 &u = raw[k][i / 4];
        const uint32_t w = (i & 3) == 0 ? u.x : (i & 3) == 1 ? u.y : (i & 3) == 2 ? u.z : u.w;
        f[i] = __uint_as_float(w);
      }
    }
    // IEEE fp32, product and sum each rounded (no FMA contraction): reading A4
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < PER_LANE; ++i) s = __fadd_rn(s, __fmul_rn(f[i], f[i]));
    s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 8));
    s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
    s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
    s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
    if (lane16 == 0 && rows[k] < bh_rows) {
      const float key = s;
      const int64_t o = b * bh_rows + rows[k];
      keys[o] = key;
      if (keys_user) keys_user[o] = key;
    }
  }
}

cudaError_t launch_norm_keys(int dtype, int d, const void *x, const int64_t *st, int64_t batch,
                             int64_t heads, int64_t L, float *keys, float *keys_user,
                             cudaStream_t stream) {
  const int64_t rows = heads * L;
  const int64_t halfwarps = (rows + kNormRows - 1) / kNormRows;
  dim3 grid((unsigned)((halfwarps * 16 + 255) / 256), (unsigned)batch);
  if (dtype == 0 && d == 128)
    norm_keys_kernel<__nv_bfloat16, 128><<<grid, 256, 0, stream>>>((const __nv_bfloat16 *)x, st[0], st[1], st[2], heads, L, keys, keys_user);
  else if (dtype == 0 && d == 64)
    norm_keys_kernel<__nv_bfloat16, 64><<<grid, 256, 0, stream>>>((const __nv_bfloat16 *)x, st[0], st[1], st[2], heads, L, keys, keys_user);
  else if (dtype == 1 && d == 128)
    norm_keys_kernel<float, 128><<<grid, 256, 0, stream>>>((const float *)x, st[0], st[1], st[2], heads, L, keys, keys_user);
  else
    norm_keys_kernel<float, 64><<<grid, 256, 0, stream>>>((const float *)x, st[0], st[1], st[2], heads, L, keys, keys_user);
  return cudaGetLastError();
}

// =====================================================================================
// K2: segmented stable LSD radix sort.
// =====================================================================================
struct TileLoc {
  int side;
  int64_t seg;        // global segment id
  int64_t seg_start;  // element offset of the segment in the combined buffer
  int64_t seg_len;
  int64_t tile_off;   // offset of this tile inside the segment
  int64_t count;      // items in this tile (may be <= 0 for empty tail tiles)
  int64_t head;       // (batch*H) index within the side
  int64_t win_start;  // token index of the window start inside the head row
};

BA_DEVICE TileLoc locate_tile(const SortGeom &g, int64_t t) {
  TileLoc r;
  int s = (g.n_sides == 2 && t >= g.side[1].tile_base) ? 1 : 0;
  const SortSide &sd = g.side[s];
  const int64_t lt = t - sd.tile_base;
  const int64_t per_head = sd.n_win * sd.tiles_per_win;
  const int64_t head = lt / per_head;
  const int64_t rem = lt - head * per_head;
  const int64_t w = rem / sd.tiles_per_win;
  const int64_t tw = rem - w * sd.tiles_per_win;
  r.side = s;
  r.head = head;
  r.seg = sd.seg_base + head * sd.n_win + w;
  r.win_start = w * sd.win;
  r.seg_start = sd.base + head * sd.L + r.win_start;
  r.seg_len = imin64(sd.win, sd.L - r.win_start);
  r.tile_off = tw * kSortTile;
  r.count = imin64(kSortTile, r.seg_len - r.tile_off);
  return r;
}

// Per-tile 256-bin histogram of digit `shift`.
__global__ void __launch_bounds__(kSortThreads) radix_hist_kernel(SortGeom g, const uint32_t *__restrict__ keys,
                                                                  uint32_t *__restrict__ hist, int shift) {
  __shared__ uint32_t h[256];
  const int64_t t = blockIdx.x;
  h[threadIdx.x] = 0;
  __syncthreads();
  const TileLoc loc = locate_tile(g, t);
  const uint32_t *src = keys + loc.seg_start + loc.tile_off;
  uint32_t kv[kSortIPT];  // all loads in flight first
#pragma unroll
  for (int r = 0; r < kSortIPT; ++r) {
    const int64_t i = threadIdx.x + (int64_t)r * kSortThreads;
    kv[r] = i < loc.count ? __ldg(src + i) : 0u;
  }
#pragma unroll
  for (int r = 0; r < kSortIPT; ++r)
    if (threadIdx.x + (int64_t)r * kSortThreads < loc.count) atomicAdd(&h[(kv[r] >> shift) & 255u], 1u);
  __syncthreads();
  hist[t * 256 + threadIdx.x] = h[threadIdx.x];
}

// Per segment: offsets[tile][digit] = sum_{d' < digit} total(d') + sum_{tile' < tile} count(tile', digit)
// (digit-major order => stable).  One CTA of 256 threads per segment; thread = digit.
__global__ void __launch_bounds__(256) radix_scan_kernel(SortGeom g, uint32_t *__restrict__ hist) {
  __shared__ uint32_t tot[256];
  const int64_t seg = blockIdx.x;
  const int s = (g.n_sides == 2 && seg >= g.side[1].seg_base) ? 1 : 0;
  const SortSide &sd = g.side[s];
  const int64_t tile0 = sd.tile_base + (seg - sd.seg_base) * sd.tiles_per_win;
  const int digit = threadIdx.x;
  uint32_t run = 0;
  for (int64_t i = 0; i < sd.tiles_per_win; ++i) {
    uint32_t c = hist[(tile0 + i) * 256 + digit];
    hist[(tile0 + i) * 256 + digit] = run;  // exclusive within digit
    run += c;
  }
  tot[digit] = run;
  __syncthreads();
  // exclusive scan of tot over digits (Hillis-Steele in smem; 256 entries)
  uint32_t v = tot[digit];
  for (int off = 1; off < 256; off <<= 1) {
    __syncthreads();
    uint32_t a = digit >= off ? tot[digit - off] : 0u;
    __syncthreads();
    tot[digit] += a;
  }
  __syncthreads();
  const uint32_t base = tot[digit] - v;
  for (int64_t i = 0; i < sd.tiles_per_win; ++i) hist[(tile0 + i) * 256 + digit] += base;
}

// Stable scatter of one tile.  Warp w owns tile items [w*512, (w+1)*512); in
// round r lane l holds item w*512 + r*32 + l.  Rank of an item among equal
// digits = (items of earlier warps) + (earlier rounds of this warp) +
// (lower lanes of this round) — exactly the original order within the tile.
template <bool kFirst, bool kLast>
__global__ void __launch_bounds__(kSortThreads) radix_scatter_kernel(
    SortGeom g, const uint32_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
    uint32_t *__restrict__ keys_out, uint32_t *__restrict__ vals_out, const uint32_t *__restrict__ offsets,
    int shift) {
  constexpr int kWarps = kSortThreads / 32;
  constexpr int kPerWarp = kSortTile / kWarps;  // 512
  __shared__ uint32_t wcount[kWarps][256];
  __shared__ uint32_t dstart[256];
  __shared__ uint32_t s_off[256];
  __shared__ uint32_t s_keys[kSortTile];
  __shared__ uint32_t s_vals[kSortTile];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = blockIdx.x;
  const TileLoc loc = locate_tile(g, t);
  if (loc.count <= 0) return;  // uniform across the CTA
  for (int i = threadIdx.x; i < kWarps * 256; i += kSortThreads) (&wcount[0][0])[i] = 0;
  s_off[threadIdx.x] = offsets[t * 256 + threadIdx.x];
  __syncthreads();

  const int64_t base = loc.seg_start + loc.tile_off;
  uint32_t key[kSortIPT], val[kSortIPT], rank[kSortIPT];
  const unsigned lt = lanemask_lt();
  // every global load in flight before the ranking rounds (their smem atomics and
  // __syncwarp would otherwise serialise one load latency per round)
#pragma unroll
  for (int r = 0; r < kSortIPT; ++r) {
    const int item = warp * kPerWarp + r * 32 + lane;
    const bool valid = item < loc.count;
    key[r] = valid ? __ldg(keys_in + base + item) : 0xffffffffu;
    if constexpr (kFirst) val[r] = (uint32_t)(loc.win_start + loc.tile_off + item);
    else val[r] = valid ? __ldg(vals_in + base + item) : 0u;
  }
#pragma unroll
  for (int r = 0; r < kSortIPT; ++r) {
    const int item = warp * kPerWarp + r * 32 + lane;
    const bool valid = item < loc.count;
    const uint32_t digit = (key[r] >> shift) & 255u;
    const unsigned vmask = __ballot_sync(0xffffffffu, valid);
    rank[r] = 0;
    if (valid) {
      const unsigned peers = __match_any_sync(vmask, digit);
      const uint32_t before = wcount[warp][digit];
      rank[r] = before + __popc(peers & lt);
      // the highest peer lane publishes the new count after all peers read it
      __syncwarp(vmask);
      if ((peers >> lane) == 1u) wcount[warp][digit] = before + __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
  {  // per digit: exclusive over warps, then tile totals
    const int dg = threadIdx.x;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = wcount[w][dg];
      wcount[w][dg] = run;
      run += c;
    }
    dstart[dg] = run;
  }
  __syncthreads();
  {  // exclusive scan of tile digit totals -> dstart
    const int dg = threadIdx.x;
    const uint32_t v = dstart[dg];
    for (int off = 1; off < 256; off <<= 1) {
      __syncthreads();
      const uint32_t a = dg >= off ? dstart[dg - off] : 0u;
      __syncthreads();
      dstart[dg] += a;
    }
    __syncthreads();
    dstart[dg] -= v;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSortIPT; ++r) {
    const int item = warp * kPerWarp + r * 32 + lane;
    if (item < loc.count) {
      const uint32_t digit = (key[r] >> shift) & 255u;
      const uint32_t pos = dstart[digit] + wcount[warp][digit] + rank[r];
      s_keys[pos] = key[r];
      s_vals[pos] = val[r];
    }
  }
  __syncthreads();
  // coalesced write-out: runs of equal digits go to consecutive global slots
  for (int i = threadIdx.x; i < loc.count; i += kSortThreads) {
    const uint32_t k = s_keys[i];
    const uint32_t digit = (k >> shift) & 255u;
    const int64_t gpos = s_off[digit] + (i - dstart[digit]);
    if constexpr (kLast) {
      const SortSide &sd = g.side[loc.side];
      sd.perm_out[loc.head * sd.L + loc.win_start + gpos] = (int32_t)s_vals[i];
    } else {
      keys_out[loc.seg_start + gpos] = k;
      vals_out[loc.seg_start + gpos] = s_vals[i];
    }
  }
}

cudaError_t launch_radix_sort(const SortGeom &g, uint32_t *keys_a, uint32_t *vals_a, uint32_t *keys_b,
                              uint32_t *vals_b, uint32_t *hist, cudaStream_t st, int *launches) {
  if (g.tiles_total == 0) return cudaSuccess;
  uint32_t *kin = keys_a, *vin = vals_a, *kout = keys_b, *vout = vals_b;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = pass * 8;
    radix_hist_kernel<<<(unsigned)g.tiles_total, kSortThreads, 0, st>>>(g, kin, hist, shift);
    radix_scan_kernel<<<(unsigned)g.segs_total, 256, 0, st>>>(g, hist);
    if (pass == 0)
      radix_scatter_kernel<true, false><<<(unsigned)g.tiles_total, kSortThreads, 0, st>>>(g, kin, vin, kout, vout, hist, shift);
    else if (pass == 3)
      radix_scatter_kernel<false, true><<<(unsigned)g.tiles_total, kSortThreads, 0, st>>>(g, kin, vin, kout, vout, hist, shift);
    else
      radix_scatter_kernel<false, false><<<(unsigned)g.tiles_total, kSortThreads, 0, st>>>(g, kin, vin, kout, vout, hist, shift);
    *launches += 3;
    uint32_t *tk = kin, *tv = vin;
    kin = kout; vin = vout; kout = tk; vout = tv;
  }
  return cudaGetLastError();
}

// =====================================================================================
// K1 + K2 in 1 + 4 launches ("onesweep", decoupled look-back):
//   keys_hist_kernel   the norm keys of K1 (same arithmetic, reading A4) for every
//                      sorted side, written to the key buffer, plus the per-segment
//                      histograms of all four 8-bit digits (smem, flushed with one
//                      atomic per non-zero bin);
//   onesweep_kernel    one stable LSD pass per digit: a tile takes a ticket (tiles
//                      therefore start in order), ranks its 4096 keys as before,
//                      publishes its per-digit counts, sums its predecessors' counts
//                      by looking back over their published (aggregate | inclusive)
//                      words, and scatters through smem (coalesced runs).  The
//                      segment's digit base comes from the histograms of the first
//                      kernel, so no separate histogram / scan launches are needed.
// Control block, zeroed by one memset per call (robust against any stale workspace
// content): seg_hist [segs][4][256] u32, status [4][tiles][256] u64, tickets [4] u32.
// =====================================================================================
constexpr int kKeysRowsPerCta = 512;    // 16 half-warps x 32 rows
constexpr uint64_t kStAgg = 1ull << 62, kStInc = 1ull << 63, kStVal = (1ull << 62) - 1;

BA_DEVICE int64_t seg_of(const SortSide &sd, int64_t head, int64_t t) { return sd.seg_base + head * sd.n_win + t / sd.win; }
BA_DEVICE uint32_t lane_id() { return threadIdx.x & 31u; }

// Row layout: FOUR lanes per row, lane l holding the chunks of A4's virtual lanes l, l+4,
// l+8, l+12 (chunk = D/16 features).  Each virtual lane's sum is sequential as in A4; the
// halving tree's first two levels (p[i] + p[i+8], then q[i] + q[i+4]) are lane-local and
// the last two are xor shuffles, so every key is bit-identical to the 16-lane form (IEEE
// addition commutes).  A warp holds 8 rows per step, so the per-row work (tree, key store,
// histogram) costs a quarter of the 16-lane layout's issue slots.
template <typename T, int D>
#ifndef BA_KEYS_RIF
#define BA_KEYS_RIF 2
#endif
#ifndef BA_KEYS_MINB
#define BA_KEYS_MINB 3
#endif
BA_DEVICE void keys_hist_chunk(const SortGeom &g, const KeysArgs &ka, float *__restrict__ keys,
                                uint32_t *__restrict__ seg_hist, int64_t c) {
  constexpr int CHUNK = D / 16;                        // features per virtual lane
  constexpr int CB = CHUNK * (int)sizeof(T);           // bytes per chunk: 8, 16 or 32
  constexpr int NV = CB >= 16 ? CB / 16 : 1;           // 16-byte loads per chunk (8-byte chunk: one uint2)
  constexpr int kRowsInFlight = NV >= 2 ? 1 : BA_KEYS_RIF;  // rows per lane per step (4 chunks each; 128 B in flight)
  constexpr int kRowsPerStep = 8 * kRowsInFlight;      // per warp
  __shared__ uint32_t hist[2][4][256];  // the chunk's first two segments
  __shared__ int64_t s_seg0;
  // chunk c -> (side, head row, chunk of kKeysRowsPerCta tokens)
  const int64_t chunks0 = g.side[0].heads * ((g.side[0].L + kKeysRowsPerCta - 1) / kKeysRowsPerCta);
  const bool s1 = g.n_sides == 2 && c >= chunks0;
  if (s1) c -= chunks0;
  // the side's fields by value (a dynamically indexed kernel-parameter array goes to local memory)
  SortSide sd;
  sd.heads = s1 ? g.side[1].heads : g.side[0].heads;
  sd.L = s1 ? g.side[1].L : g.side[0].L;
  sd.win = s1 ? g.side[1].win : g.side[0].win;
  sd.n_win = s1 ? g.side[1].n_win : g.side[0].n_win;
  sd.base = s1 ? g.side[1].base : g.side[0].base;
  sd.seg_base = s1 ? g.side[1].seg_base : g.side[0].seg_base;
  const int64_t cph = (sd.L + kKeysRowsPerCta - 1) / kKeysRowsPerCta;
  const int64_t head = c / cph, t0 = (c - head * cph) * kKeysRowsPerCta;
  const int nrow = (int)imin64(kKeysRowsPerCta, sd.L - t0);
  const T *x = static_cast<const T *>(s1 ? ka.x[1] : ka.x[0]);
  const int64_t stv0 = s1 ? ka.st[1][0] : ka.st[0][0], stv1 = s1 ? ka.st[1][1] : ka.st[0][1],
                stv2 = s1 ? ka.st[1][2] : ka.st[0][2];
  float *user = s1 ? ka.user[1] : ka.user[0];
  const int64_t H = sd.heads / ka.batch, bb = head / H, hh = head - bb * H;
  for (int i = threadIdx.x; i < 2 * 4 * 256; i += 256) (&hist[0][0][0])[i] = 0u;
  if (threadIdx.x == 0) s_seg0 = seg_of(sd, head, t0);
  __syncthreads();
  const int64_t seg0 = s_seg0;
  // segment of row t relative to seg0 without a per-row 64-bit division: a chunk spans at
  // most two windows of >= kKeysRowsPerCta tokens (boundary b1); tiny windows divide in 32 bits
  const int64_t w0 = t0 / sd.win, b1 = (w0 + 1) * sd.win;
  const bool tiny_win = sd.win < kKeysRowsPerCta;
  const uint32_t win32 = (uint32_t)imin64(sd.win, 0x7fffffff);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, l4 = lane & 3, rsub = lane >> 2;
  const T *xbase = x + bb * stv0 + hh * stv1 + t0 * stv2 + l4 * CHUNK;
  constexpr int kRowsPerWarp = kKeysRowsPerCta / 8;  // 64
  for (int it = 0; it < kRowsPerWarp / kRowsPerStep; ++it) {
    uint4 raw[kRowsInFlight][4][NV];
    int rr[kRowsInFlight];
#pragma unroll
    for (int k = 0; k < kRowsInFlight; ++k) {  // every load first
      const int r = warp * kRowsPerWarp + it * kRowsPerStep + k * 8 + rsub;
      rr[k] = r;
      if (r < nrow) {
        const T *p = xbase + (int64_t)r * stv2;
#pragma unroll
        for (int v = 0; v < 4; ++v) {  // virtual lane l4 + 4v: features [(l4 + 4v) * CHUNK, +CHUNK)
          const T *pc = p + v * 4 * CHUNK;
          if constexpr (CB == 8) {
            const uint2 u = __ldg(reinterpret_cast<const uint2 *>(pc));
            raw[k][v][0] = make_uint4(u.x, u.y, 0, 0);
          } else {
#pragma unroll
            for (int n = 0; n < NV; ++n) raw[k][v][n] = ldg16(pc + n * (16 / (int)sizeof(T)));
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kRowsInFlight; ++k) {
      float pv[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        float f[CHUNK];
        if constexpr (sizeof(T) == 2) {
#pragma unroll
          for (int i = 0; i < CHUNK / 2; ++i) {
            const uint4 &u = raw[k][v][i / 4];
            const uint32_t w = (i & 3) == 0 ? u.x : (i & 3) == 1 ? u.y : (i & 3) == 2 ? u.z : u.w;
            f[2 * i] = __uint_as_float(w << 16);
            f[2 * i + 1] = __uint_as_float(w & 0xffff0000u);
          }
        } else {
#pragma unroll
          for (int i = 0; i < CHUNK; ++i) {
            const uint4 &u = raw[k][v][i / 4];
            const uint32_t w = (i & 3) == 0 ? u.x : (i & 3) == 1 ? u.y : (i & 3) == 2 ? u.z : u.w;
            f[i] = __uint_as_float(w);
          }
        }
        // IEEE fp32, product and sum each rounded (no FMA contraction): reading A4
        float sv = 0.f;
#pragma unroll
        for (int i = 0; i < CHUNK; ++i) sv = __fadd_rn(sv, __fmul_rn(f[i], f[i]));
        pv[v] = sv;
      }
      // halving tree: p[i] + p[i+8] (v, v+2), q[i] + q[i+4] (v = 0, 1), then r[i] + r[i+2], s[0] + s[1]
      float s = __fadd_rn(__fadd_rn(pv[0], pv[2]), __fadd_rn(pv[1], pv[3]));
      s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
      s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
      const bool ok = rr[k] < nrow;
      const int64_t t = t0 + rr[k];
      if (ok && l4 == 0) {
        keys[sd.base + head * sd.L + t] = s;
        if (user) user[head * sd.L + t] = s;
      }
      // histograms: lane l4 of each row takes digit l4; lanes with equal (segment, digit, value)
      // are aggregated first (match_any: the high digits of similar keys collide on a few bins)
      const int64_t sg = !ok ? 0 : !tiny_win ? (int64_t)(t >= b1) : (int64_t)((uint32_t)(t - w0 * sd.win) / win32);
      const uint32_t dg = (__float_as_uint(s) >> (8 * l4)) & 255u;
      const unsigned amask = __ballot_sync(0xffffffffu, ok);
      if (ok) {
        const uint32_t tag = ((uint32_t)l4 << 8 | dg) + (sg < 2 ? (uint32_t)sg << 10 : 0x80000000u + lane);
        const unsigned peers = __match_any_sync(amask, tag);
        if ((peers & lanemask_lt()) == 0) {  // the lowest lane of each group adds the group's count
          if (sg < 2) atomicAdd(&hist[sg][l4][dg], (uint32_t)__popc(peers));
          else atomicAdd(&seg_hist[(seg0 + sg) * 1024 + l4 * 256 + dg], 1u);  // tiny windows only
        }
      }
    }
  }
  __syncthreads();
  const int64_t seg1 = seg_of(sd, head, t0 + nrow - 1);
  for (int i = threadIdx.x; i < 2 * 1024; i += 256) {
    const int sg = i >> 10;
    if (seg0 + sg > seg1) break;
    const uint32_t v = (&hist[sg][0][0])[i & 1023];
    if (v) atomicAdd(&seg_hist[(seg0 + sg) * 1024 + (i & 1023)], v);
  }
  __syncthreads();  // hist / s_seg0 are reused by the CTA's next chunk
}

// K1 as one persistent cooperative launch: the CTAs first zero the sort's control block
// (segment histograms, look-back status, tickets; no stale workspace content survives), one
// grid-wide barrier, then grid-stride over the 512-row chunks — the memset this replaces
// was a launch of its own.
template <typename T, int D>
__global__ void __launch_bounds__(256, BA_KEYS_MINB) keys_hist_kernel(SortGeom g, KeysArgs ka, float *__restrict__ keys,
                                                                      uint32_t *__restrict__ seg_hist, uint4 *__restrict__ ctrl,
                                                                      int64_t ctrl_words, int64_t n_chunks) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ctrl_words; i += (int64_t)gridDim.x * blockDim.x)
    ctrl[i] = make_uint4(0u, 0u, 0u, 0u);
  __threadfence();
  cooperative_groups::this_grid().sync();
  for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) keys_hist_chunk<T, D>(g, ka, keys, seg_hist, c);
}

BA_DEVICE uint64_t ld_status(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
BA_DEVICE void st_status(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// One stable LSD pass (digit `pass`) over every segment: see the block comment above.
template <bool kFirst, bool kLast>
__global__ void __launch_bounds__(kSortThreads) onesweep_kernel(
    SortGeom g, const uint32_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
    uint32_t *__restrict__ keys_out, uint32_t *__restrict__ vals_out, const uint32_t *__restrict__ seg_hist,
    uint64_t *__restrict__ status, uint32_t *__restrict__ tickets, int pass) {
  constexpr int kWarps = kSortThreads / 32;
  constexpr int kPerWarp = kSortTile / kWarps;  // 512
  __shared__ uint32_t wcount[kWarps][256];
  __shared__ uint32_t dstart[256];
  __shared__ uint32_t s_off[256];
  __shared__ uint32_t s_keys[kSortTile];
  __shared__ uint32_t s_vals[kSortTile];
  __shared__ uint32_t s_ticket;
  __shared__ uint32_t wsum[kWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) s_ticket = atomicAdd(tickets + pass, 1u);  // tiles start in ticket order
  __syncthreads();
  const int64_t t = s_ticket;
  const TileLoc loc = locate_tile(g, t);
  if (loc.count <= 0) return;  // empty tail tile of a window: nobody looks back at it
  const int shift = 8 * pass;
  for (int i = threadIdx.x; i < kWarps * 256; i += kSortThreads) (&wcount[0][0])[i] = 0;
  __syncthreads();

  const int64_t base = loc.seg_start + loc.tile_off;
  uint32_t key[kSortIPT], val[kSortIPT], rank[kSortIPT];
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < kSortIPT; ++r) {
    const int item = warp * kPerWarp + r * 32 + lane;
    const bool valid = item < loc.count;
    key[r] = valid ? __ldg(keys_in + base + item) : 0xffffffffu;
    if constexpr (kFirst) val[r] = (uint32_t)(loc.win_start + loc.tile_off + item);
    else val[r] = valid ? __ldg(vals_in + base + item) : 0u;
  }
#pragma unroll
  for (int r = 0; r < kSortIPT; ++r) {
    const int item = warp * kPerWarp + r * 32 + lane;
    const bool valid = item < loc.count;
    const uint32_t digit = (key[r] >> shift) & 255u;
    const unsigned vmask = __ballot_sync(0xffffffffu, valid);
    rank[r] = 0;
    if (valid) {
      const unsigned peers = __match_any_sync(vmask, digit);
      const uint32_t before = wcount[warp][digit];
      rank[r] = before + __popc(peers & lt);
      __syncwarp(vmask);
      if ((peers >> lane) == 1u) wcount[warp][digit] = before + __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
  const int dg = threadIdx.x;  // one thread per digit from here
  uint32_t cnt;
  {  // per digit: exclusive over warps, then the tile's count
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = wcount[w][dg];
      wcount[w][dg] = run;
      run += c;
    }
    cnt = run;
  }
  // publish this tile's count, then look back over the segment's earlier tiles
  uint64_t *st_pass = status + (int64_t)pass * g.tiles_total * 256;
  const int64_t tile_in_seg = loc.tile_off / kSortTile;
  uint64_t prefix = 0;
  if (tile_in_seg == 0) {
    st_status(st_pass + t * 256 + dg, kStInc | cnt);
  } else {
    st_status(st_pass + t * 256 + dg, kStAgg | cnt);
    for (int64_t j = t - 1;; --j) {
      uint64_t v;
      do { v = ld_status(st_pass + j * 256 + dg); } while (!(v & (kStAgg | kStInc)));
      prefix += v & kStVal;
      if (v & kStInc) break;
    }
    st_status(st_pass + t * 256 + dg, kStInc | (prefix + cnt));
  }
  // exclusive scans over the 256 digits (one per thread): shuffle scan within each warp, then
  // the totals of the lower warps (2 barriers per scan instead of 16)
  auto exscan256 = [&](uint32_t v) -> uint32_t {
    uint32_t x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    uint32_t wpre = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) wpre += w < warp ? wsum[w] : 0u;
    __syncthreads();  // wsum is reused by the next scan
    return wpre + x - v;
  };
  // the segment's digit base: exclusive scan of its histogram over the digits; global position of
  // this tile's first digit-dg item
  s_off[dg] = exscan256(seg_hist[loc.seg * 1024 + pass * 256 + dg]) + (uint32_t)prefix;
  dstart[dg] = exscan256(cnt);  // tile-local digit starts
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSortIPT; ++r) {
    const int item = warp * kPerWarp + r * 32 + lane;
    if (item < loc.count) {
      const uint32_t digit = (key[r] >> shift) & 255u;
      const uint32_t pos = dstart[digit] + wcount[warp][digit] + rank[r];
      s_keys[pos] = key[r];
      s_vals[pos] = val[r];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < loc.count; i += kSortThreads) {
    const uint32_t k = s_keys[i];
    const uint32_t digit = (k >> shift) & 255u;
    const int64_t gpos = s_off[digit] + (i - dstart[digit]);
    if constexpr (kLast) {
      const SortSide &sd = g.side[loc.side];
      sd.perm_out[loc.head * sd.L + loc.win_start + gpos] = (int32_t)s_vals[i];
    } else {
      keys_out[loc.seg_start + gpos] = k;
      vals_out[loc.seg_start + gpos] = s_vals[i];
    }
  }
}

size_t sort_ctrl_bytes(const SortGeom &g) {
  return (size_t)g.segs_total * 1024 * 4 + (size_t)4 * g.tiles_total * 256 * 8 + 64;
}

cudaError_t launch_keys_sort(const SortGeom &g, int dtype, int d, const KeysArgs &ka, uint32_t *keys_a,
                             uint32_t *vals_a, uint32_t *keys_b, uint32_t *vals_b, void *ctrl, cudaStream_t st,
                             int *launches) {
  if (g.tiles_total == 0) return cudaSuccess;
  uint32_t *seg_hist = static_cast<uint32_t *>(ctrl);
  uint64_t *status = reinterpret_cast<uint64_t *>(static_cast<char *>(ctrl) + (size_t)g.segs_total * 1024 * 4);
  uint32_t *tickets = reinterpret_cast<uint32_t *>(status + (size_t)4 * g.tiles_total * 256);
  int64_t chunks = 0;
  for (int s = 0; s < g.n_sides; ++s) chunks += g.side[s].heads * ((g.side[s].L + kKeysRowsPerCta - 1) / kKeysRowsPerCta);
  void *kernel = dtype == 0 ? (d == 128 ? (void *)keys_hist_kernel<__nv_bfloat16, 128> : (void *)keys_hist_kernel<__nv_bfloat16, 64>)
                            : (d == 128 ? (void *)keys_hist_kernel<float, 128> : (void *)keys_hist_kernel<float, 64>);
  int per_sm = 0, dev = 0, sms = 0;
  cudaError_t e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, 0)) != cudaSuccess) return e;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorLaunchOutOfResources;
  const unsigned kgrid = (unsigned)std::min<int64_t>(chunks, (int64_t)per_sm * sms);
  float *keys_f = reinterpret_cast<float *>(keys_a);
  uint4 *ctrl16 = static_cast<uint4 *>(ctrl);
  int64_t ctrl_words = (int64_t)((sort_ctrl_bytes(g) + 15) / 16);
  SortGeom gg = g;
  KeysArgs kk = ka;
  void *kargs[] = {&gg, &kk, &keys_f, &seg_hist, &ctrl16, &ctrl_words, &chunks};
  if ((e = cudaLaunchCooperativeKernel(kernel, dim3(kgrid), dim3(256), kargs, 0, st)) != cudaSuccess) return e;
  uint32_t *kin = keys_a, *vin = vals_a, *kout = keys_b, *vout = vals_b;
  for (int pass = 0; pass < 4; ++pass) {
    const unsigned grid = (unsigned)g.tiles_total;
    if (pass == 0)
      onesweep_kernel<true, false><<<grid, kSortThreads, 0, st>>>(g, kin, vin, kout, vout, seg_hist, status, tickets, pass);
    else if (pass == 3)
      onesweep_kernel<false, true><<<grid, kSortThreads, 0, st>>>(g, kin, vin, kout, vout, seg_hist, status, tickets, pass);
    else
      onesweep_kernel<false, false><<<grid, kSortThreads, 0, st>>>(g, kin, vin, kout, vout, seg_hist, status, tickets, pass);
    uint32_t *tk = kin, *tv = vin;
    kin = kout; vin = vout; kout = tk; vout = tv;
  }
  *launches += 5;  // keys/histograms (zeroing the control block first) + 4 passes
  return cudaGetLastError();
}

// =====================================================================================
// K3: gather rows through pi and compute per-block mean / population variance.
// One CTA (256 threads) per (block g, batch*head).  A thread owns one 16-byte
// chunk (EPC features) of rows r0, r0 + RPI, ...: every row load is in flight
// before the copies are stored.  The moments are ONE pass over the registers
// with a per-column shift K = the block's first row (exact in fp64):
//   mean = K + S1/n,  var = S2/n - (S1/n)^2,  S1 = sum (x - K), S2 = sum (x - K)^2
// — one fp32 -> fp64 conversion per element (the conversions run on the XU pipe,
// which the two-pass form saturated), and the shift keeps the cancellation at
// eps * (var + (mean - K)^2) instead of eps * (var + mean^2).
// =====================================================================================
template <typename T, int D, int NBLK = 1>
BA_DEVICE void gather_stats_body(const T *__restrict__ x, int64_t s0, int64_t s1, int64_t s2, int64_t heads, int64_t L,
                                 int B, const int32_t *__restrict__ perm, int32_t *__restrict__ perm_id_out,
                                 T *__restrict__ xs, double *__restrict__ mean, double *__restrict__ var, int64_t gp,
                                 int64_t bh) {
  // NBLK blocks per CTA (NBLK * B <= 128 rows): B = 64 runs two blocks per CTA so that as
  // many row loads are in flight per SM as at B = 128; the moments are per block
  constexpr int EPC = Chunk<T>::EPC;
  constexpr int CPR = D / EPC;       // chunks per row
  constexpr int RPI = 256 / CPR;     // rows per iteration
  constexpr int MAXIT = 128 / RPI;   // NBLK * B <= 128
  static_assert(CPR * 2 == 32 || CPR == 32 || CPR * 4 == 32, "row groups per warp");
  constexpr int GPW = 32 / CPR;                 // row groups per warp (combined by shuffles)
  constexpr int RG = RPI / GPW;                 // partial rows left for the smem reduction
  __shared__ double red[2][RG][D + 1];
  __shared__ double s_shift[D];
  const int64_t b = bh / heads, h = bh - b * heads;  // gp: block group, bh: batch * heads + head
  const int chunk = threadIdx.x % CPR;
  const int rsub = threadIdx.x / CPR;
  const int64_t row0 = gp * NBLK * B;
  const int n = (int)imin64((int64_t)NBLK * B, L - row0);
  const T *xbase = x + b * s0 + h * s1 + chunk * EPC;
  T *xsbase = xs ? xs + (bh * L + row0) * D + chunk * EPC : nullptr;
  // stage 1: source row indices; stage 2: every row load in flight; stage 3: stores + sums
  int32_t src[MAXIT];  // L < 2^31 (validated)
#pragma unroll
  for (int it = 0; it < MAXIT; ++it) {
    const int r = rsub + it * RPI;
    src[it] = -1;
    if (r < n) {
      const int64_t tok = row0 + r;
      if (perm) {
        src[it] = __ldg(perm + bh * L + tok);
      } else {
        src[it] = (int32_t)tok;
        if (perm_id_out && chunk == 0) perm_id_out[bh * L + tok] = (int32_t)tok;
      }
    }
  }
  uint4 raw[MAXIT];
#pragma unroll
  for (int it = 0; it < MAXIT; ++it)
    raw[it] = src[it] >= 0 ? ldg16(xbase + (int64_t)src[it] * s2) : make_uint4(0, 0, 0, 0);
  // shift row of the first block = its first row (loaded before the copy stores, like the rows)
  uint4 kraw0 = make_uint4(0, 0, 0, 0);
  if (mean) kraw0 = ldg16(xbase + (int64_t)(perm ? __ldg(perm + bh * L + row0) : (int32_t)row0) * s2);
  if (xs) {  // permuted copy (NULL: zero-copy attention reads the rows through pi itself)
#pragma unroll
    for (int it = 0; it < MAXIT; ++it) {
      const int r = rsub + it * RPI;
      if (r < n) stg16(xsbase + (int64_t)r * D, raw[it]);
    }
  }
  if (!mean) return;  // V: copy only
  const int64_t nb = (L + B - 1) / B;
#pragma unroll 1
  for (int sb = 0; sb < NBLK; ++sb) {
    const int64_t g = gp * NBLK + sb;
    if (g >= nb) break;  // CTA-uniform
    const int r_lo = sb * B;
    const int nsb = (int)imin64(B, L - g * B);
    if (sb > 0) __syncthreads();  // red / s_shift reuse
    // shift row = the block's first row
    const uint4 kraw = sb == 0 ? kraw0 : ldg16(xbase + (int64_t)(perm ? __ldg(perm + bh * L + g * B) : (int32_t)(g * B)) * s2);
    double kc[EPC], a1[EPC], a2[EPC];
    {
      float v[EPC];
      Chunk<T>::unpack(kraw, v);
#pragma unroll
      for (int e = 0; e < EPC; ++e) { kc[e] = (double)v[e]; a1[e] = 0.0; a2[e] = 0.0; }
    }
#pragma unroll
    for (int it = 0; it < MAXIT; ++it) {
      const int r = rsub + it * RPI;
      if (r >= r_lo && r < r_lo + nsb) {
        float v[EPC];
        Chunk<T>::unpack(raw[it], v);
#pragma unroll
        for (int e = 0; e < EPC; ++e) {
          const double dv = (double)v[e] - kc[e];
          a1[e] += dv;
          a2[e] = fma(dv, dv, a2[e]);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < EPC; ++e) {
#pragma unroll
      for (int off = CPR; off < 32; off <<= 1) {
        a1[e] += __shfl_xor_sync(0xffffffffu, a1[e], off);
        a2[e] += __shfl_xor_sync(0xffffffffu, a2[e], off);
      }
    }
    if ((threadIdx.x & 31) < CPR) {
#pragma unroll
      for (int e = 0; e < EPC; ++e) { red[0][rsub / GPW][chunk * EPC + e] = a1[e]; red[1][rsub / GPW][chunk * EPC + e] = a2[e]; }
    }
    if (rsub == 0) {
#pragma unroll
      for (int e = 0; e < EPC; ++e) s_shift[chunk * EPC + e] = kc[e];
    }
    __syncthreads();
    const double inv_n = 1.0 / (double)nsb;
    for (int c = threadIdx.x; c < D; c += 256) {
      double t1 = 0.0, t2 = 0.0;
#pragma unroll
      for (int i = 0; i < RG; ++i) { t1 += red[0][i][c]; t2 += red[1][i][c]; }
      const double m1 = t1 * inv_n;
      mean[(bh * nb + g) * D + c] = s_shift[c] + m1;
      var[(bh * nb + g) * D + c] = fmax(fma(-m1, m1, t2 * inv_n), 0.0);
    }
  }
}

template <typename T, int D>
__global__ void __launch_bounds__(256, 3) gather_stats_kernel(
    const T *__restrict__ x, int64_t s0, int64_t s1, int64_t s2, int64_t heads, int64_t L, int B,
    const int32_t *__restrict__ perm, int32_t *__restrict__ perm_id_out, T *__restrict__ xs,
    double *__restrict__ mean, double *__restrict__ var) {
  gather_stats_body<T, D>(x, s0, s1, s2, heads, L, B, perm, perm_id_out, xs, mean, var, blockIdx.x, blockIdx.y);
}

// Q, K and V of one ba_select in ONE launch (one CTA per (side, block, batch*head),
// sides laid out back to back in a 1-D grid): no inter-kernel drain between them.
template <typename T, int D, int NBLK>
__global__ void __launch_bounds__(256, 3) gather_stats_multi_kernel(const GatherSides gs, int B) {
  int64_t c = blockIdx.x;
  int s = 0;
  while (s + 1 < gs.n && c >= gs.side[s].ctas) { c -= gs.side[s].ctas; ++s; }
  const GatherSide &sd = gs.side[s];
  const int64_t ng = ((sd.L + B - 1) / B + NBLK - 1) / NBLK;  // block groups per (batch, head)
  gather_stats_body<T, D, NBLK>(static_cast<const T *>(sd.x), sd.st[0], sd.st[1], sd.st[2], sd.heads, sd.L, B, sd.perm,
                                sd.perm_id_out, static_cast<T *>(sd.xs), sd.mean, sd.var, c % ng, c / ng);
}

cudaError_t launch_gather_stats_multi(int dtype, int d, GatherSides gs, int B, cudaStream_t stream) {
  const int nblk = B <= 64 ? 2 : 1;  // B = 64: two blocks per CTA (128 rows in flight)
  int64_t total = 0;
  for (int s = 0; s < gs.n; ++s) {
    gs.side[s].ctas = (((gs.side[s].L + B - 1) / B + nblk - 1) / nblk) * gs.side[s].heads * gs.side[s].batch;
    total += gs.side[s].ctas;
  }
  if (total == 0) return cudaSuccess;
  // heads in gather_stats_body index one batch element's heads; bh runs over batch * heads
#define BA_GM(T, D)                                                                     \
  do {                                                                                  \
    if (nblk == 2) gather_stats_multi_kernel<T, D, 2><<<(unsigned)total, 256, 0, stream>>>(gs, B); \
    else gather_stats_multi_kernel<T, D, 1><<<(unsigned)total, 256, 0, stream>>>(gs, B);           \
  } while (0)
  if (dtype == 0 && d == 128) BA_GM(__nv_bfloat16, 128);
  else if (dtype == 0 && d == 64) BA_GM(__nv_bfloat16, 64);
  else if (dtype == 1 && d == 128) BA_GM(float, 128);
  else BA_GM(float, 64);
#undef BA_GM
  return cudaGetLastError();
}

cudaError_t launch_gather_stats(int dtype, int d, const void *x, const int64_t *st, int64_t batch,
                                int64_t heads, int64_t L, int B, const int32_t *perm,
                                int32_t *perm_id_out, void *xs, double *mean, double *var,
                                cudaStream_t stream) {
  dim3 grid((unsigned)((L + B - 1) / B), (unsigned)(batch * heads));
#define BA_GS(T, D) gather_stats_kernel<T, D><<<grid, 256, 0, stream>>>((const T *)x, st[0], st[1], st[2], heads, L, B, perm, perm_id_out, (T *)xs, mean, var)
  if (dtype == 0 && d == 128) BA_GS(__nv_bfloat16, 128);
  else if (dtype == 0 && d == 64) BA_GS(__nv_bfloat16, 64);
  else if (dtype == 1 && d == 128) BA_GS(float, 128);
  else BA_GS(float, 64);
#undef BA_GS
  return cudaGetLastError();
}

// =====================================================================================
// K3b (NEXT-4): per-block covariance Sigma_g = (1/n) sum_i (x_i - xbar)(x_i - xbar)^T
// in fp64 for the exact compensation tr(SigmaQ SigmaK)/d (Eq. cov-comp,
// P:494-495).  One CTA (256 threads) per (block, batch*head); rows are read through
// pi (like K3) 16 at a time, centred in fp64 into smem, and each thread accumulates
// a (D/16) x (D/16) patch: rows ty + 16 i, columns tx + 16 j (conflict-free reads).
// =====================================================================================
template <typename T, int D>
__global__ void __launch_bounds__(256) block_cov_kernel(const T *__restrict__ x, int64_t s0, int64_t s1, int64_t s2,
                                                        int64_t heads, int64_t L, int B, const int32_t *__restrict__ perm,
                                                        const double *__restrict__ mean, double *__restrict__ cov) {
  constexpr int R = D / 16;
  constexpr int EPC = Chunk<T>::EPC, CPR = D / EPC, RPC = 256 / CPR;  // rows per load pass
  constexpr int CH = 16;                                               // rows per smem chunk
  __shared__ double xc[CH][D + 1];
  __shared__ double mu[D];
  const int64_t g = blockIdx.x, bh = blockIdx.y;
  const int64_t b = bh / heads, h = bh - b * heads;
  const int64_t nb = (L + B - 1) / B;
  const int64_t row0 = g * B;
  const int n = (int)imin64(B, L - row0);
  for (int c = threadIdx.x; c < D; c += 256) mu[c] = mean[(bh * nb + g) * D + c];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[R][R];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < R; ++j) acc[i][j] = 0.0;
  const T *xbase = x + b * s0 + h * s1;
  const int chunk = threadIdx.x % CPR, rsub = threadIdx.x / CPR;
  __syncthreads();
  for (int r0 = 0; r0 < n; r0 += CH) {
    for (int rr = rsub; rr < CH; rr += RPC) {
      const int r = r0 + rr;
      float v[EPC];
      if (r < n) {
        const int64_t tok = row0 + r;
        const int64_t src = perm ? (int64_t)__ldg(perm + bh * L + tok) : tok;
        Chunk<T>::unpack(ldg16(xbase + src * s2 + chunk * EPC), v);
      }
#pragma unroll
      for (int e = 0; e < EPC; ++e) xc[rr][chunk * EPC + e] = r < n ? (double)v[e] - mu[chunk * EPC + e] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = 0; rr < CH; ++rr) {
      double a[R], c2[R];
#pragma unroll
      for (int i = 0; i < R; ++i) { a[i] = xc[rr][ty + 16 * i]; c2[i] = xc[rr][tx + 16 * i]; }
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int j = 0; j < R; ++j) acc[i][j] = fma(a[i], c2[j], acc[i][j]);
    }
    __syncthreads();
  }
  const double inv_n = 1.0 / (double)n;
  double *out = cov + (bh * nb + g) * (int64_t)D * D;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < R; ++j) out[(ty + 16 * i) * D + tx + 16 * j] = acc[i][j] * inv_n;
}

cudaError_t launch_block_cov(int dtype, int d, const void *x, const int64_t *st, int64_t batch, int64_t heads, int64_t L,
                             int B, const int32_t *perm, const double *mean, double *cov, cudaStream_t stream) {
  dim3 grid((unsigned)((L + B - 1) / B), (unsigned)(batch * heads));
#define BA_BC(T, D) block_cov_kernel<T, D><<<grid, 256, 0, stream>>>((const T *)x, st[0], st[1], st[2], heads, L, B, perm, mean, cov)
  if (dtype == 0 && d == 128) BA_BC(__nv_bfloat16, 128);
  else if (dtype == 0 && d == 64) BA_BC(__nv_bfloat16, 64);
  else if (dtype == 1 && d == 128) BA_BC(float, 128);
  else BA_BC(float, 64);
#undef BA_BC
  return cudaGetLastError();
}

// =====================================================================================
// K4a: compensated block logits as an fp64 micro-GEMM over 3d features.
// =====================================================================================
constexpr int kScK = 8;  // features per smem stage

// TILE x TILE output tile, 256 threads as a 16 x 16 grid, (TILE/16)^2 outputs per
// thread: rows ty + 16 i and columns tx + 16 j — a warp's 16 column threads read
// 16 consecutive doubles (128 B: every bank once) and its two row groups are
// broadcasts, so the smem operand reads are conflict-free (the former
// tx*4 + j mapping put 4 threads on each bank pair).  TILE = 64 for small score
// maps (config A: 128 tiles of 128 would leave SMs idle).
template <int D, int TILE>
__global__ void __launch_bounds__(256) scores_kernel(int64_t hq, int64_t grp, int64_t nq, int64_t nk,
                                                     const double *__restrict__ q_mean,
                                                     const double *__restrict__ q_var,
                                                     const double *__restrict__ k_mean,
                                                     const double *__restrict__ k_var, int comp,
                                                     double inv_sqrt_d, double beta_over_d,
                                                     double *__restrict__ logits) {
  constexpr int R = TILE / 16;              // outputs per thread per dim
  constexpr int LPT = TILE * kScK / 256;    // features each thread loads per operand per stage
  constexpr int TPR = kScK / LPT;           // loader threads per row
  __shared__ __align__(16) double As[2][kScK][TILE + 2];
  __shared__ __align__(16) double Bs[2][kScK][TILE + 2];
  const int64_t bhq = blockIdx.z;            // batch * hq + head
  const int64_t b = bhq / hq, h = bhq - b * hq;
  const int64_t bhk = b * (hq / grp) + h / grp;
  const int64_t gq0 = (int64_t)blockIdx.y * TILE, gk0 = (int64_t)blockIdx.x * TILE;
  const double *qm = q_mean + bhq * nq * D, *qv = q_var + bhq * nq * D;
  const double *km = k_mean + bhk * nk * D, *kv = k_var + bhk * nk * D;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[R][R];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < R; ++j) acc[i][j] = 0.0;
  const int nfeat = comp ? 3 * D : D;
  // loader: thread -> (row = tid / TPR, LPT features); features of part p at column t:
  //   Xq = [Qbar/sqrt(d), (beta/d) VarQ, (beta/d) Qbar^2],  Xk = [Kbar, Kbar^2 + VarK, VarK]
  // Register-staged prefetch: the next stage's global loads are issued before the
  // current stage's FMAs and stored to smem after them, so their latency is hidden.
  const int lr = threadIdx.x / TPR, lf = (threadIdx.x % TPR) * LPT;
  const int64_t gq_l = gq0 + lr, gk_l = gk0 + lr;
  const bool q_ok = gq_l < nq, k_ok = gk_l < nk;
  double rqm[LPT], rqv[LPT], rkm[LPT], rkv[LPT];
  auto fetch = [&](int c0) {
#pragma unroll
    for (int e = 0; e < LPT; ++e) {
      const int c = c0 + lf + e;
      const int part = c / D, t = c - part * D;
      rqm[e] = q_ok ? qm[gq_l * D + t] : 0.0;
      rqv[e] = (q_ok && part == 1) ? qv[gq_l * D + t] : 0.0;
      rkm[e] = (k_ok && part < 2) ? km[gk_l * D + t] : 0.0;
      rkv[e] = (k_ok && part > 0) ? kv[gk_l * D + t] : 0.0;
    }
  };
  auto stash = [&](int c0, int buf) {
#pragma unroll
    for (int e = 0; e < LPT; ++e) {
      const int c = c0 + lf + e;
      const int part = c / D;
      const double m = rqm[e], k = rkm[e];
      As[buf][lf + e][lr] = part == 0 ? m * inv_sqrt_d : part == 1 ? beta_over_d * rqv[e] : beta_over_d * (m * m);
      Bs[buf][lf + e][lr] = part == 0 ? k : part == 1 ? fma(k, k, rkv[e]) : rkv[e];
    }
  };
  fetch(0);
  stash(0, 0);
  __syncthreads();
  int buf = 0;
  for (int c0 = 0; c0 < nfeat; c0 += kScK) {
    const bool more = c0 + kScK < nfeat;
    if (more) fetch(c0 + kScK);  // loads in flight during the FMAs below
#pragma unroll
    for (int k = 0; k < kScK; ++k) {
      double a[R], bb[R];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        a[i] = As[buf][k][ty + 16 * i];
        bb[i] = Bs[buf][k][tx + 16 * i];
      }
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int j = 0; j < R; ++j) acc[i][j] = fma(a[i], bb[j], acc[i][j]);
    }
    if (more) stash(c0 + kScK, buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int64_t gq = gq0 + ty + 16 * i;
    if (gq >= nq) continue;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int64_t gk = gk0 + tx + 16 * j;
      if (gk < nk) logits[(bhq * nq + gq) * nk + gk] = acc[i][j];
    }
  }
}

constexpr int kScoresKS = 8;   // features per smem stage of the DMMA kernel (32: register and smem budget exceeded)

// The same inner product of length 3d on the FP64 tensor path: mma.sync
// m8n8k4.f64 (DMMA).  Measured on B200 (tools/dmma_bench.cu) DMMA and DFMA both
// peak at 128 FLOP/clk/SM, but one DMMA does the work of 8 warp-wide DFMAs per
// 2 operand loads, so the issue slots and smem reads that held the SIMT kernel
// to ~39% of peak stop binding.  CTA tile TILE x TILE, warps of 32 x 32 (4 x 4
// DMMA tiles, 32 fp64 accumulators per thread), KS features per stage (KS/4
// k-steps of 4), register-staged prefetch of the next stage.
// Fragments (PTX m8n8k4 .f64): g = lane/4, t = lane%4;  A[g][t], B[t][g],
// C[g][2t + {0,1}].
// kExact (NEXT-4, Eq. cov-comp): l' = Qbar.Kbar/sqrt(d) + (beta/d) tr(SigmaQ SigmaK)
// = one inner product of length d + d^2 with Xq = [Qbar/sqrt(d), (beta/d) vec SigmaQ] and
// Xk = [Kbar, vec SigmaK] (the covariances are symmetric: tr(AB) = vec(A).vec(B));
// q_var / k_var then point at the covariances [.., N, d, d].
template <int TILE, int KS>
struct ScoresSmem {
  static constexpr int LDS = TILE + 8;  // k-row stride (doubles): 4 k-rows -> 2 wavefronts
  double A[2][KS][LDS];
  double B[2][KS][LDS];
};

// One TILE x TILE tile of l' (query blocks gq0.., key blocks gk0.. of q-head bhq) on the
// FP64 tensor path; the CTA's (TILE/32)^2 warps, operands staged through sm.
template <int D, int TILE, int KS, bool kExact>
BA_DEVICE void scores_tile(int64_t hq, int64_t grp, int64_t nq, int64_t nk, const double *__restrict__ q_mean,
                           const double *__restrict__ q_var, const double *__restrict__ k_mean,
                           const double *__restrict__ k_var, int comp, double inv_sqrt_d, double beta_over_d,
                           double *__restrict__ logits, int64_t bhq, int64_t gq0, int64_t gk0,
                           ScoresSmem<TILE, KS> &sm) {
  constexpr int WARPS = (TILE / 32) * (TILE / 32), NT = WARPS * 32;
  constexpr int LPT = TILE * KS / NT;               // features each thread loads per operand per stage
  constexpr int TPR = KS / LPT;                     // loader threads per row
  auto &As = sm.A;
  auto &Bs = sm.B;
  const int64_t b = bhq / hq, h = bhq - b * hq;
  const int64_t bhk = b * (hq / grp) + h / grp;
  constexpr int64_t VW = kExact ? D * D : D;  // per-block width of q_var / k_var
  const double *qm = q_mean + bhq * nq * D, *qv = q_var + bhq * nq * VW;
  const double *km = k_mean + bhk * nk * D, *kv = k_var + bhk * nk * VW;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = (warp / (TILE / 32)) * 32, wc = (warp % (TILE / 32)) * 32;  // warp tile origin
  const int g = lane >> 2, tq = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int nfeat = kExact ? D + D * D : comp ? 3 * D : D;
  const int lr = threadIdx.x / TPR, lf = (threadIdx.x % TPR) * LPT;
  const int64_t gq_l = gq0 + lr, gk_l = gk0 + lr;
  const bool q_ok = gq_l < nq, k_ok = gk_l < nk;
  double rqm[LPT], rqv[LPT], rkm[LPT], rkv[LPT];
  auto fetch = [&](int c0) {
#pragma unroll
    for (int e2 = 0; e2 < LPT; ++e2) {
      const int c = c0 + lf + e2;
      if constexpr (kExact) {  // c < D: the means; c >= D: vec(Sigma) entry c - D
        rqm[e2] = q_ok ? (c < D ? qm[gq_l * D + c] : qv[gq_l * VW + (c - D)]) : 0.0;
        rkm[e2] = k_ok ? (c < D ? km[gk_l * D + c] : kv[gk_l * VW + (c - D)]) : 0.0;
      } else {
        const int part = c / D, tt = c - part * D;
        rqm[e2] = q_ok ? qm[gq_l * D + tt] : 0.0;
        rqv[e2] = (q_ok && part == 1) ? qv[gq_l * D + tt] : 0.0;
        rkm[e2] = (k_ok && part < 2) ? km[gk_l * D + tt] : 0.0;
        rkv[e2] = (k_ok && part > 0) ? kv[gk_l * D + tt] : 0.0;
      }
    }
  };
  auto stash = [&](int c0, int buf) {  // Xq = [Qbar/sqrt(d), (beta/d) VarQ, (beta/d) Qbar^2], Xk = [Kbar, Kbar^2 + VarK, VarK]
#pragma unroll
    for (int e2 = 0; e2 < LPT; ++e2) {
      const int c = c0 + lf + e2;
      if constexpr (kExact) {
        As[buf][lf + e2][lr] = c < D ? rqm[e2] * inv_sqrt_d : beta_over_d * rqm[e2];
        Bs[buf][lf + e2][lr] = rkm[e2];
      } else {
        const int part = c / D;
        const double m = rqm[e2], k = rkm[e2];
        As[buf][lf + e2][lr] = part == 0 ? m * inv_sqrt_d : part == 1 ? beta_over_d * rqv[e2] : beta_over_d * (m * m);
        Bs[buf][lf + e2][lr] = part == 0 ? k : part == 1 ? fma(k, k, rkv[e2]) : rkv[e2];
      }
    }
  };
  fetch(0);
  stash(0, 0);
  __syncthreads();
  int buf = 0;
  for (int c0 = 0; c0 < nfeat; c0 += KS) {
    const bool more = c0 + KS < nfeat;
    if (more) fetch(c0 + KS);
#pragma unroll
    for (int k4 = 0; k4 < KS; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        af[i] = As[buf][k4 + tq][wr + 8 * i + g];
        bf[i] = Bs[buf][k4 + tq][wc + 8 * i + g];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(acc[i][j][0]), "+d"(acc[i][j][1])
                       : "d"(af[i]), "d"(bf[j]));
    }
    if (more) stash(c0 + KS, buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gq = gq0 + wr + 8 * i + g;
    if (gq >= nq) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gk = gk0 + wc + 8 * j + 2 * tq;
      double *dst = logits + (bhq * nq + gq) * nk + gk;
      if (gk + 1 < nk && ((nk & 1) == 0)) {
        *reinterpret_cast<double2 *>(dst) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else {
        if (gk < nk) dst[0] = acc[i][j][0];
        if (gk + 1 < nk) dst[1] = acc[i][j][1];
      }
    }
  }
}

// The diagonal-compensation tile with fewer, larger warp tiles (K4a, default): 8 warps of
// 32 x 64 outputs (4 x 8 DMMA tiles, 64 fp64 accumulators per thread), 16 features per smem
// stage (4 k-steps, half the CTA barriers of the 32 x 32 / 8-feature form), the next
// k-step's fragments loaded while the current k-step's 32 DMMAs issue, and per stage only
// the operand arrays that stage's feature part needs (a stage never straddles a part).
// Measured (ncu, config A) the 32 x 32 form stalled on smem fragment latency (short
// scoreboard 19%) and barriers (14%) as much as on the FP64 pipe (20%).
constexpr int kScW_KS = 16, kScW_LDS = 128 + 4;  // +4: the 4 fragment rows tq of a half-warp fall on distinct bank groups
struct ScoresSmemW {
  double A[2][kScW_KS][kScW_LDS];
  double B[2][kScW_KS][kScW_LDS];
};
template <int D>
BA_DEVICE void scores_tile_w(int64_t hq, int64_t grp, int64_t nq, int64_t nk, const double *__restrict__ q_mean,
                             const double *__restrict__ q_var, const double *__restrict__ k_mean,
                             const double *__restrict__ k_var, int comp, double inv_sqrt_d, double beta_over_d,
                             double *__restrict__ logits, int64_t bhq, int64_t gq0, int64_t gk0, ScoresSmemW &sm) {
  constexpr int TILE = 128, KS = kScW_KS, LPT = TILE * KS / 256;  // 8 features per thread per operand per stage
  static_assert(D % KS == 0, "a stage never straddles a feature part");
  const int64_t b = bhq / hq, h = bhq - b * hq;
  const int64_t bhk = b * (hq / grp) + h / grp;
  const double *qm = q_mean + bhq * nq * D, *qv = q_var + bhq * nq * D;
  const double *km = k_mean + bhk * nk * D, *kv = k_var + bhk * nk * D;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = (warp >> 1) * 32, wc = (warp & 1) * 64;  // warp tile origin
  const int g = lane >> 2, tq = lane & 3;
  double acc[4][8][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int nfeat = comp ? 3 * D : D;
  const int lr = threadIdx.x >> 1, lf = (threadIdx.x & 1) * LPT;  // loader: row lr, features lf .. lf + 7
  const bool q_ok = gq0 + lr < nq, k_ok = gk0 + lr < nk;
  const double *qrow_m = qm + (gq0 + lr) * D + lf, *qrow_v = qv + (gq0 + lr) * D + lf;
  const double *krow_m = km + (gk0 + lr) * D + lf, *krow_v = kv + (gk0 + lr) * D + lf;
  double r0[LPT], r1[LPT], r2[LPT];  // part 0: qm, km; part 1: qv, km, kv; part 2: qm, kv
  auto ld8 = [](double *dst, const double *src, bool ok) {
#pragma unroll
    for (int e = 0; e < LPT; e += 2) {
      const double2 v = ok ? __ldg(reinterpret_cast<const double2 *>(src + e)) : make_double2(0.0, 0.0);
      dst[e] = v.x;
      dst[e + 1] = v.y;
    }
  };
  auto fetch = [&](int c0) {
    const int part = c0 / D, t = c0 - part * D;
    if (part == 0) { ld8(r0, qrow_m + t, q_ok); ld8(r1, krow_m + t, k_ok); }
    else if (part == 1) { ld8(r0, qrow_v + t, q_ok); ld8(r1, krow_m + t, k_ok); ld8(r2, krow_v + t, k_ok); }
    else { ld8(r0, qrow_m + t, q_ok); ld8(r2, krow_v + t, k_ok); }
  };
  auto stash = [&](int c0, int buf) {  // Xq = [Qbar/sqrt(d), (beta/d) VarQ, (beta/d) Qbar^2], Xk = [Kbar, Kbar^2 + VarK, VarK]
    const int part = c0 / D;
#pragma unroll
    for (int e = 0; e < LPT; ++e) {
      double xa, xb;
      if (part == 0) { xa = r0[e] * inv_sqrt_d; xb = r1[e]; }
      else if (part == 1) { xa = beta_over_d * r0[e]; xb = fma(r1[e], r1[e], r2[e]); }
      else { xa = beta_over_d * (r0[e] * r0[e]); xb = r2[e]; }
      sm.A[buf][lf + e][lr] = xa;
      sm.B[buf][lf + e][lr] = xb;
    }
  };
  fetch(0);
  stash(0, 0);
  __syncthreads();
  int buf = 0;
  for (int c0 = 0; c0 < nfeat; c0 += KS) {
    const bool more = c0 + KS < nfeat;
    if (more) fetch(c0 + KS);  // global loads in flight during the DMMAs below
    double af[2][4], bf[2][8];
#pragma unroll
    for (int i = 0; i < 4; ++i) af[0][i] = sm.A[buf][tq][wr + 8 * i + g];
#pragma unroll
    for (int j = 0; j < 8; ++j) bf[0][j] = sm.B[buf][tq][wc + 8 * j + g];
#pragma unroll
    for (int s4 = 0; s4 < KS / 4; ++s4) {
      const int cur = s4 & 1;
      if (s4 + 1 < KS / 4) {  // next k-step's fragments ahead of this k-step's DMMAs
#pragma unroll
        for (int i = 0; i < 4; ++i) af[cur ^ 1][i] = sm.A[buf][4 * (s4 + 1) + tq][wr + 8 * i + g];
#pragma unroll
        for (int j = 0; j < 8; ++j) bf[cur ^ 1][j] = sm.B[buf][4 * (s4 + 1) + tq][wc + 8 * j + g];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(acc[i][j][0]), "+d"(acc[i][j][1])
                       : "d"(af[cur][i]), "d"(bf[cur][j]));
    }
    if (more) stash(c0 + KS, buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gq = gq0 + wr + 8 * i + g;
    if (gq >= nq) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t gk = gk0 + wc + 8 * j + 2 * tq;
      double *dst = logits + (bhq * nq + gq) * nk + gk;
      if (gk + 1 < nk && ((nk & 1) == 0)) {
        *reinterpret_cast<double2 *>(dst) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else {
        if (gk < nk) dst[0] = acc[i][j][0];
        if (gk + 1 < nk) dst[1] = acc[i][j][1];
      }
    }
  }
}

template <int D, int TILE, int KS, bool kExact = false>
__global__ void __launch_bounds__((TILE / 32) * (TILE / 32) * 32) scores_mma_kernel(
    int64_t hq, int64_t grp, int64_t nq, int64_t nk, const double *__restrict__ q_mean,
    const double *__restrict__ q_var, const double *__restrict__ k_mean, const double *__restrict__ k_var,
    int comp, double inv_sqrt_d, double beta_over_d, double *__restrict__ logits) {
  __shared__ __align__(16) ScoresSmem<TILE, KS> sm;
  scores_tile<D, TILE, KS, kExact>(hq, grp, nq, nk, q_mean, q_var, k_mean, k_var, comp, inv_sqrt_d, beta_over_d, logits,
                                   blockIdx.z, (int64_t)blockIdx.y * TILE, (int64_t)blockIdx.x * TILE, sm);
}

cudaError_t launch_scores(int d, int64_t batch, int64_t hq, int64_t hkv, int64_t nq, int64_t nk,
                          const double *q_mean, const double *q_var, const double *k_mean,
                          const double *k_var, int comp, double beta, double *logits,
                          cudaStream_t st) {
  const double inv_sqrt_d = 1.0 / sqrt((double)d), bod = beta / (double)d;
  const int64_t grp = hq / hkv;
  // BA_SCORES_SIMT=1 selects the SIMT DFMA kernel (A/B profiling knob)
  const int64_t big = ((nk + 127) / 128) * ((nq + 127) / 128) * batch * hq;
  // 128-tiles (16 warps) unless fewer than ~100 CTAs would result (A: 128 CTAs of 128 beat 512 of 64: 0.79 -> 0.76 ms selection)
  static const int tile_min = getenv("BA_SCORES_TILE128_MIN") ? atoi(getenv("BA_SCORES_TILE128_MIN")) : 100;
  const int tile = big >= tile_min ? 128 : 64;
  static int simt = -1;
  if (simt < 0) simt = getenv("BA_SCORES_SIMT") ? atoi(getenv("BA_SCORES_SIMT")) : 0;
  dim3 grid((unsigned)((nk + tile - 1) / tile), (unsigned)((nq + tile - 1) / tile), (unsigned)(batch * hq));
  if (simt && comp != 2) {
#define BA_SC(D, T) scores_kernel<D, T><<<grid, 256, 0, st>>>(hq, grp, nq, nk, q_mean, q_var, k_mean, k_var, comp, inv_sqrt_d, bod, logits)
    if (d == 128) { if (tile == 128) BA_SC(128, 128); else BA_SC(128, 64); }
    else { if (tile == 128) BA_SC(64, 128); else BA_SC(64, 64); }
#undef BA_SC
    return cudaGetLastError();
  }
#define BA_SM(D, T, X) scores_mma_kernel<D, T, kScoresKS, X><<<grid, (T / 32) * (T / 32) * 32, 0, st>>>(hq, grp, nq, nk, q_mean, q_var, k_mean, k_var, comp, inv_sqrt_d, bod, logits)
  if (comp == 2) {  // exact covariance compensation: q_var / k_var are the block covariances
    if (d == 128) { if (tile == 128) BA_SM(128, 128, true); else BA_SM(128, 64, true); }
    else { if (tile == 128) BA_SM(64, 128, true); else BA_SM(64, 64, true); }
    return cudaGetLastError();
  }
  if (d == 128) { if (tile == 128) BA_SM(128, 128, false); else BA_SM(128, 64, false); }
  else { if (tile == 128) BA_SM(64, 128, false); else BA_SM(64, 64, false); }
#undef BA_SM
  return cudaGetLastError();
}

// =====================================================================================
// K4b: per-row top-kappa.  One warp per row; the row's l' values sit in smem.
// =====================================================================================
// Order-preserving bits of a non-negative double back to its value.
BA_DEVICE double unordered_pos(uint64_t u) { return __longlong_as_double((long long)(u ^ 0x8000000000000000ull)); }

// Warp sum in a fixed order (lane-strided sequential partials, then an xor
// tree): deterministic, so reruns give bit-identical kappa_row.
BA_DEVICE double warp_sum_det(double v) {
#pragma unroll
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// Cumulative-mass budget (reading A23, NEXT-1): kappa_row = the length of the
// shortest (-m', g_k)-ordered prefix whose mass reaches p.  u[] holds the
// order-preserving bits of m' (>= 0).  A 16-pass MSD radix select with 4-bit
// digits finds the value T of the crossing entry: per pass every lane keeps
// 16 fp64 bucket masses and counts of the candidates sharing the prefix in
// registers, reduced deterministically across the warp; the digit where the
// running mass (from the top) reaches p is kept.  Then entries > T are counted
// and summed once more, and the entries equal to T are added (ascending g_k)
// until the mass reaches p.
BA_DEVICE unsigned topp_count(const uint64_t *u, int64_t nk, double p, double total, int lane) {
  if (total < p) return (unsigned)nk;  // the whole row does not reach p: keep everything
  uint64_t T = 0, pmask = 0;
  double above = 0.0;  // mass of the entries above the current prefix range
  for (int pass = 0; pass < 16; ++pass) {
    const int shift = 60 - 4 * pass;
    double acc[16];
    unsigned cnt[16];
#pragma unroll
    for (int b = 0; b < 16; ++b) { acc[b] = 0.0; cnt[b] = 0u; }
    for (int64_t j = lane; j < nk; j += 32) {
      const uint64_t v = u[j];
      if ((v & pmask) == T) {
        const unsigned dg = (unsigned)(v >> shift) & 15u;
        const double val = unordered_pos(v);
#pragma unroll
        for (int b = 0; b < 16; ++b) {
          const bool hit = dg == (unsigned)b;
          acc[b] += hit ? val : 0.0;
          cnt[b] += hit ? 1u : 0u;
        }
      }
    }
#pragma unroll
    for (int b = 0; b < 16; ++b) {
      acc[b] = warp_sum_det(acc[b]);
      cnt[b] = __reduce_add_sync(0xffffffffu, cnt[b]);
    }
    // the crossing digit; if fp64 re-association leaves no crossing, the lowest non-empty digit
    int dsel = -1, lowest = -1;
    double run = above;
#pragma unroll
    for (int b = 15; b >= 0; --b) {
      if (!cnt[b]) continue;
      lowest = b;
      if (dsel < 0) {
        if (run + acc[b] >= p) dsel = b;
        else run += acc[b];
      }
    }
    if (dsel < 0) dsel = lowest;
#pragma unroll
    for (int b = 15; b >= 0; --b)
      if (b > dsel) above += acc[b];
    T |= (uint64_t)dsel << shift;
    pmask |= 0xFull << shift;
  }
  // exact pass: entries strictly above T, then T's ties in ascending g_k
  double s_gt = 0.0;
  unsigned c_gt = 0, c_eq = 0;
  for (int64_t j = lane; j < nk; j += 32) {
    const uint64_t v = u[j];
    if (v > T) { s_gt += unordered_pos(v); ++c_gt; }
    c_eq += v == T;
  }
  s_gt = warp_sum_det(s_gt);
  c_gt = __reduce_add_sync(0xffffffffu, c_gt);
  c_eq = __reduce_add_sync(0xffffffffu, c_eq);
  const double tv = unordered_pos(T);
  unsigned need = 0;
  double cum = s_gt;
  while (need < c_eq && cum < p) { cum += tv; ++need; }
  if (need == 0) need = 1;  // s_gt >= p only through re-association: a near-tie inside the band
  return c_gt + need;
}

// One row of K4b by one warp: x = the warp's nk doubles of smem, hist = its 256 counters.
BA_DEVICE void topk_row(int64_t row, int64_t nk, int64_t kappa, double top_p, const double *__restrict__ logits,
                        int32_t *__restrict__ kv_index, int32_t *__restrict__ kv_count, uint8_t *__restrict__ mask,
                        double *__restrict__ prob, double *__restrict__ tau, double *x, unsigned *hist) {
  const int lane = threadIdx.x & 31;
  const double *src = logits + row * nk;
  double mx = -INFINITY;
  for (int64_t j = lane; j < nk; j += 32) {
    const double v = src[j];
    x[j] = v;
    mx = fmax(mx, v);
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  __syncwarp();
  double denom = 0.0, total = 0.0;
  const bool topp = top_p > 0.0;
  const bool need_prob = (prob != nullptr) || (tau != nullptr) || topp;
  if (need_prob) {
    for (int64_t j = lane; j < nk; j += 32) denom += exp(x[j] - mx);
#pragma unroll
    for (int off = 16; off; off >>= 1) denom += __shfl_xor_sync(0xffffffffu, denom, off);
    if (topp) {  // rank by m' itself (reading A23 orders by (-m', g_k))
      for (int64_t j = lane; j < nk; j += 32) {
        const double mp = exp(x[j] - mx) / denom;
        x[j] = mp;
        total += mp;
        if (prob) prob[row * nk + j] = mp;
      }
      total = warp_sum_det(total);
    } else if (prob) {
      for (int64_t j = lane; j < nk; j += 32) prob[row * nk + j] = exp(x[j] - mx) / denom;
    }
  }
  // kappa-th largest ordered key by an 8-pass MSD radix select (8-bit digits):
  // per pass, histogram the digit of the candidates sharing the current prefix
  // (per-warp smem histogram), then pick the digit holding the k_rem-th largest.
  for (int64_t j = lane; j < nk; j += 32)
    reinterpret_cast<uint64_t *>(x)[j] = ordered_bits(x[j]);  // in place: keys from here on
  __syncwarp();
  const uint64_t *u = reinterpret_cast<const uint64_t *>(x);
  uint64_t T = 0, pmask = 0;
  unsigned k_rem = (unsigned)kappa;  // TOPK: kappa; TOPP: min(kappa_row, kappa) (kappa = the density cap)
  if (topp) {
    const unsigned kp = topp_count(u, nk, top_p, total, lane);
    if (kp < k_rem) k_rem = kp;
  }
  const unsigned k_row = k_rem;
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
#pragma unroll
    for (int i = 0; i < 8; ++i) hist[lane * 8 + i] = 0;
    __syncwarp();
    for (int64_t j = lane; j < nk; j += 32) {
      const uint64_t v = u[j];
      if ((v & pmask) == T) atomicAdd(&hist[(v >> shift) & 255u], 1u);
    }
    __syncwarp();
    // lane owns digits [8*lane, 8*lane + 8); suffix sums from the top digit down
    unsigned c[8], tot = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) { c[i] = hist[lane * 8 + i]; tot += c[i]; }
    unsigned above = tot;  // inclusive suffix over lanes >= lane
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned o = __shfl_down_sync(0xffffffffu, above, off);
      if (lane + off < 32) above += o;
    }
    above -= tot;  // candidates in digits owned by higher lanes
    int dsel = -1;
    unsigned before = 0;
    unsigned run = above;
#pragma unroll
    for (int i = 7; i >= 0; --i) {
      if (dsel < 0 && run < k_rem && run + c[i] >= k_rem) { dsel = lane * 8 + i; before = run; }
      run += c[i];
    }
    const unsigned ball = __ballot_sync(0xffffffffu, dsel >= 0);
    const int owner = __ffs(ball) - 1;
    const unsigned c_bin = hist[dsel < 0 ? 0 : dsel];  // read before the shuffle (owner's dsel is valid)
    dsel = __shfl_sync(0xffffffffu, dsel, owner);
    before = __shfl_sync(0xffffffffu, before, owner);
    const unsigned n_bin = __shfl_sync(0xffffffffu, c_bin, owner);  // candidates sharing the new prefix
    k_rem -= before;
    T |= (uint64_t)dsel << shift;
    pmask |= 0xFFull << shift;
    __syncwarp();
    if (pass < 7 && n_bin <= 32) {
      // at most 32 candidates left: one per lane, and the k_rem-th largest of them is T, found by
      // counting, for each, the candidates above it (the same T and tie count the remaining radix
      // passes would reach)
      uint64_t *cs = reinterpret_cast<uint64_t *>(hist);  // this pass's histogram is consumed: 128 slots
      unsigned base_n = 0;
      for (int64_t j0 = 0; j0 < nk && base_n < n_bin; j0 += 32) {  // warp-uniform bound
        const int64_t j = j0 + lane;
        const uint64_t v = j < nk ? u[j] : 0ull;
        const bool in = j < nk && (v & pmask) == T;
        const unsigned m = __ballot_sync(0xffffffffu, in);
        if (in) cs[base_n + __popc(m & lanemask_lt())] = v;
        base_n += __popc(m);
      }
      __syncwarp();
      const bool have = (unsigned)lane < n_bin;
      const uint64_t cand = have ? cs[lane] : 0ull;
      __syncwarp();
      unsigned gt = 0, ge = 0;
#pragma unroll 1
      for (int i = 0; i < (int)n_bin; ++i) {
        const uint64_t o = __shfl_sync(0xffffffffu, cand, i);
        gt += o > cand;
        ge += o >= cand;
      }
      const bool is_t = have && gt < k_rem && k_rem <= ge;
      const unsigned tb = __ballot_sync(0xffffffffu, is_t);
      const int tl = __ffs(tb) - 1;
      T = __shfl_sync(0xffffffffu, cand, tl);
      k_rem -= __shfl_sync(0xffffffffu, gt, tl);
      break;
    }
  }
  const unsigned need_eq = k_rem;  // equal-to-T entries still needed (>= 1); the rest are > T
  unsigned eq_seen = 0, sel_seen = 0;
  const unsigned lt = lanemask_lt();
  for (int64_t j0 = 0; j0 < nk; j0 += 32) {
    const int64_t j = j0 + lane;
    bool sel = false, eq = false;
    if (j < nk) {
      const uint64_t v = u[j];
      eq = (v == T);
      sel = v > T;
    }
    const unsigned eqm = __ballot_sync(0xffffffffu, eq);
    if (eq) sel = (eq_seen + __popc(eqm & lt)) < need_eq;
    const unsigned selm = __ballot_sync(0xffffffffu, sel);
    if (sel) kv_index[row * kappa + sel_seen + __popc(selm & lt)] = (int32_t)j;
    if (mask && j < nk) mask[row * nk + j] = sel ? 1 : 0;
    eq_seen += __popc(eqm);
    sel_seen += __popc(selm);
  }
  if (lane == 0) kv_count[row] = (int32_t)k_row;
  if (tau && lane == 0) {
    // invert the order-preserving map: T holds the kappa-th largest l' (TOPP: m') exactly
    const uint64_t tb = (T >> 63) ? (T ^ 0x8000000000000000ull) : ~T;
    const double tval = __longlong_as_double((long long)tb);
    tau[row] = topp ? tval : exp(tval - mx) / denom;
  }
}

__global__ void topk_kernel(int64_t rows, int64_t nk, int64_t kappa, double top_p, const double *__restrict__ logits,
                            int32_t *__restrict__ kv_index, int32_t *__restrict__ kv_count,
                            uint8_t *__restrict__ mask, double *__restrict__ prob,
                            double *__restrict__ tau) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  unsigned *hist_base = reinterpret_cast<unsigned *>(smem_raw + (size_t)(blockDim.x >> 5) * nk * sizeof(double));
  if (row >= rows) return;
  topk_row(row, nk, kappa, top_p, logits, kv_index, kv_count, mask, prob, tau,
           reinterpret_cast<double *>(smem_raw) + (int64_t)warp * nk, hist_base + warp * 256);
}

// K4a + K4b in ONE cooperative launch: every CTA first computes l' tiles (grid-strided over
// the (key tile, query tile, q-head) space, 16 warps per 128 x 128 tile), the grid
// synchronises once, and then every warp selects rows (grid-strided) — the top-kappa needs
// complete rows, hence the grid-wide barrier.  Shared memory: the score tiles' operand
// stages, reused by the top-kappa rows afterwards.
template <int D, bool kExact, bool kWide>
__global__ void __launch_bounds__(kWide ? 256 : 512, 1) scores_topk_kernel(int64_t hq, int64_t grp, int64_t nq, int64_t nk,
                                                            const double *__restrict__ q_mean,
                                                            const double *__restrict__ q_var,
                                                            const double *__restrict__ k_mean,
                                                            const double *__restrict__ k_var, int comp,
                                                            double inv_sqrt_d, double beta_over_d,
                                                            double *__restrict__ logits, int64_t bh_total,
                                                            int64_t kappa, double top_p, int32_t *__restrict__ kv_index,
                                                            int32_t *__restrict__ kv_count, uint8_t *__restrict__ mask,
                                                            double *__restrict__ prob, double *__restrict__ tau,
                                                            int topk_warps) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t tq = (nq + 127) / 128, tk = (nk + 127) / 128;
  const int64_t tiles = tq * tk * bh_total;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t bhq = t / (tq * tk), r = t - bhq * tq * tk, iq = r / tk, ik = r - iq * tk;
    if constexpr (kWide)
      scores_tile_w<D>(hq, grp, nq, nk, q_mean, q_var, k_mean, k_var, comp, inv_sqrt_d, beta_over_d, logits, bhq,
                       iq * 128, ik * 128, *reinterpret_cast<ScoresSmemW *>(smem_raw));
    else
      scores_tile<D, 128, kScoresKS, kExact>(hq, grp, nq, nk, q_mean, q_var, k_mean, k_var, comp, inv_sqrt_d, beta_over_d,
                                             logits, bhq, iq * 128, ik * 128,
                                             *reinterpret_cast<ScoresSmem<128, kScoresKS> *>(smem_raw));
    __syncthreads();  // the operand stages are reused by the next tile
  }
  __threadfence();
  cooperative_groups::this_grid().sync();
  const int warp = threadIdx.x >> 5;
  if (warp >= topk_warps) return;
  unsigned *hist_base = reinterpret_cast<unsigned *>(smem_raw + (size_t)topk_warps * nk * sizeof(double));
  double *x = reinterpret_cast<double *>(smem_raw) + (int64_t)warp * nk;
  const int64_t rows = bh_total * nq;
  for (int64_t row = (int64_t)blockIdx.x * topk_warps + warp; row < rows; row += (int64_t)gridDim.x * topk_warps)
    topk_row(row, nk, kappa, top_p, logits, kv_index, kv_count, mask, prob, tau, x, hist_base + warp * 256);
}

cudaError_t launch_topk(int64_t rows, int64_t nk, int64_t kappa, double top_p, const double *logits,
                        int32_t *kv_index, int32_t *kv_count, uint8_t *mask, double *prob, double *tau,
                        cudaStream_t st);

cudaError_t launch_scores_topk(int d, int64_t batch, int64_t hq, int64_t hkv, int64_t nq, int64_t nk,
                               const double *q_mean, const double *q_var, const double *k_mean, const double *k_var,
                               int comp, double beta, double *logits, int64_t kappa, double top_p, int32_t *kv_index,
                               int32_t *kv_count, uint8_t *mask, double *prob, double *tau, cudaStream_t st, int *launches) {
  const double inv_sqrt_d = 1.0 / sqrt((double)d), bod = beta / (double)d;
  int64_t grp = hq / hkv, bh_total = batch * hq;
  constexpr size_t kMaxSmem = 227 * 1024;
  // the wide-tile DMMA form (8 warps) for the diagonal / no compensation; the exact
  // covariance form keeps the 16-warp 32 x 32 tiles (BA_SCORES_NARROW=1: A/B knob)
  static int narrow = -1;
  if (narrow < 0) narrow = getenv("BA_SCORES_NARROW") ? atoi(getenv("BA_SCORES_NARROW")) : 0;
  const bool wide = comp != 2 && !narrow;
  const int threads = wide ? 256 : 512;
  const size_t per_warp = (size_t)nk * sizeof(double) + 256 * sizeof(unsigned);
  int topk_warps = (int)std::min<size_t>(threads / 32, kMaxSmem / per_warp);
  if (topk_warps < 1) return cudaErrorInvalidValue;  // N_k beyond the shared-memory row buffer (validated earlier)
  size_t smem = std::max(wide ? sizeof(ScoresSmemW) : sizeof(ScoresSmem<128, kScoresKS>), (size_t)topk_warps * per_warp);
  void *kernel;
  if (comp == 2) kernel = d == 128 ? (void *)scores_topk_kernel<128, true, false> : (void *)scores_topk_kernel<64, true, false>;
  else if (wide) kernel = d == 128 ? (void *)scores_topk_kernel<128, false, true> : (void *)scores_topk_kernel<64, false, true>;
  else kernel = d == 128 ? (void *)scores_topk_kernel<128, false, false> : (void *)scores_topk_kernel<64, false, false>;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0, dev = 0, sms = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem)) != cudaSuccess) return e;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorLaunchOutOfResources;
  const int64_t tiles = ((nq + 127) / 128) * ((nk + 127) / 128) * bh_total;
  const int64_t rows_per_pass = (int64_t)topk_warps;
  int64_t want = std::max<int64_t>(tiles, (bh_total * nq + rows_per_pass - 1) / rows_per_pass);
  const unsigned grid = (unsigned)std::min<int64_t>(want, (int64_t)per_sm * sms);
  double kap_d = 0;
  (void)kap_d;
  // The top-kappa rows run as their own launch by default: after the grid barrier the fused
  // phase had one 8-warp CTA per SM and was latency-bound (C: selection 3.32 -> 3.02 ms, A
  // 0.717 -> 0.699 ms split; profiles/round2_k4_split.json).  BA_K4_SPLIT=0: fused (A/B knob).
  static int split = -1;
  if (split < 0) split = getenv("BA_K4_SPLIT") ? atoi(getenv("BA_K4_SPLIT")) : 1;
  int tw = split ? 0 : topk_warps;
  void *args[] = {&hq, &grp, &nq, &nk, (void *)&q_mean, (void *)&q_var, (void *)&k_mean, (void *)&k_var, &comp,
                  (void *)&inv_sqrt_d, (void *)&bod, &logits, &bh_total, &kappa, &top_p, &kv_index, &kv_count, &mask,
                  &prob, &tau, &tw};
  e = cudaLaunchCooperativeKernel(kernel, dim3(grid), dim3(threads), args, smem, st);
  if (launches) ++*launches;
  if (e != cudaSuccess || !split) return e;
  if (launches) ++*launches;
  return launch_topk(bh_total * nq, nk, kappa, top_p, logits, kv_index, kv_count, mask, prob, tau, st);
}

cudaError_t launch_topk(int64_t rows, int64_t nk, int64_t kappa, double top_p, const double *logits,
                        int32_t *kv_index, int32_t *kv_count, uint8_t *mask, double *prob, double *tau,
                        cudaStream_t st) {
  int warps = 8;
  while (warps > 1 && (size_t)warps * (nk * sizeof(double) + 1024) > 160 * 1024) warps >>= 1;
  const size_t smem = (size_t)warps * (nk * sizeof(double) + 256 * sizeof(unsigned));
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const unsigned grid = (unsigned)((rows + warps - 1) / warps);
  topk_kernel<<<grid, warps * 32, smem, st>>>(rows, nk, kappa, top_p, logits, kv_index, kv_count, mask, prob, tau);
  return cudaGetLastError();
}

}  // namespace baatt
