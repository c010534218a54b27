// kernels.h — internal launch interface between api.cu and the kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifdef __CUDACC__
#define BA_HOST_DEVICE_INLINE __host__ __device__ __forceinline__
#else
#define BA_HOST_DEVICE_INLINE inline
#endif

namespace baatt {

// ---------------------------------------------------------------- sort geometry
// A "side" is Q or K.  Every (batch, head) row of length L is split into
// windows of `win` tokens (win = L for the global sort); every window is one
// independently sorted segment; every segment is cut into tiles of kSortTile.
constexpr int kSortThreads = 256;
constexpr int kSortIPT = 16;
constexpr int kSortTile = kSortThreads * kSortIPT;  // 4096 keys per tile

struct SortSide {
  int64_t heads = 0;          // batch * H
  int64_t L = 0;
  int64_t win = 0;            // window length (== L for global)
  int64_t n_win = 0;          // ceil(L / win)
  int64_t tiles_per_win = 0;  // ceil(win / kSortTile)
  int64_t base = 0;           // element offset of this side in the combined key buffer
  int64_t tile_base = 0;      // first global tile id of this side
  int64_t seg_base = 0;       // first global segment id of this side
  int32_t *perm_out = nullptr;
  int64_t tiles() const { return heads * n_win * tiles_per_win; }
  int64_t segs() const { return heads * n_win; }
};

struct SortGeom {
  SortSide side[2];
  int n_sides = 0;
  int64_t tiles_total = 0;
  int64_t segs_total = 0;
  int64_t keys_total = 0;
};

// ---------------------------------------------------------------- K1 .. K4
// dtype: 0 = bf16, 1 = fp32
cudaError_t launch_norm_keys(int dtype, int d, const void *x, const int64_t *stride, int64_t batch,
                             int64_t heads, int64_t L, float *keys, float *keys_user,
                             cudaStream_t st);
cudaError_t launch_radix_sort(const SortGeom &g, uint32_t *keys_a, uint32_t *vals_a, uint32_t *keys_b,
                              uint32_t *vals_b, uint32_t *hist, cudaStream_t st, int *launches);
// K1 + K2 fused into 1 + 4 launches (+ 1 memset of the control block): the norm keys of the
// sorted sides with their per-segment digit histograms, then four onesweep passes.
// Side s of the SortGeom reads ka.x[s] with strides ka.st[s]; ka.user[s] (or NULL) gets a
// copy of the keys in original order.
struct KeysArgs {
  const void *x[2];
  int64_t st[2][3];
  float *user[2];
  int64_t batch;
};
size_t sort_ctrl_bytes(const SortGeom &g);
// ctrl: sort_ctrl_bytes(g) of workspace, zeroed here by one memset per call.
cudaError_t launch_keys_sort(const SortGeom &g, int dtype, int d, const KeysArgs &ka, uint32_t *keys_a,
                             uint32_t *vals_a, uint32_t *keys_b, uint32_t *vals_b, void *ctrl, cudaStream_t st,
                             int *launches);
cudaError_t launch_gather_stats(int dtype, int d, const void *x, const int64_t *stride, int64_t batch,
                                int64_t heads, int64_t L, int B, const int32_t *perm,
                                int32_t *perm_identity_out, void *xs, double *mean, double *var,
                                cudaStream_t st);
// NEXT-4: per-block covariance [b, H, N, d, d] fp64 of the rows x[pi] (perm NULL = identity)
cudaError_t launch_block_cov(int dtype, int d, const void *x, const int64_t *stride, int64_t batch, int64_t heads,
                             int64_t L, int B, const int32_t *perm, const double *mean, double *cov, cudaStream_t st);
// comp: 0 none, 1 diagonal (q_var / k_var = variances), 2 exact (q_var / k_var = covariances)
// K3 for several tensors (Q, K, V) in one launch
struct GatherSide {
  const void *x;
  int64_t st[3];
  int64_t batch, heads, L;
  const int32_t *perm;      // nullptr = identity
  int32_t *perm_id_out;     // identity permutation written here when perm == nullptr (or nullptr)
  void *xs;                 // permuted copy or nullptr
  double *mean, *var;       // nullptr = copy only
  int64_t ctas;             // filled by the launcher
};
struct GatherSides {
  GatherSide side[3];
  int n = 0;
};
cudaError_t launch_gather_stats_multi(int dtype, int d, GatherSides gs, int B, cudaStream_t st);
cudaError_t launch_scores(int d, int64_t batch, int64_t hq, int64_t hkv, int64_t nq, int64_t nk,
                          const double *q_mean, const double *q_var, const double *k_mean,
                          const double *k_var, int comp, double beta, double *logits,
                          cudaStream_t st);
// largest N_k the top-kappa kernel takes: one warp holds a row of N_k fp64 logits (+1 KB of
// histograms) in shared memory (227 KB per CTA)
constexpr int64_t kSelectMaxNk = 28672;
// K4a + K4b in one cooperative launch (grid-wide barrier between the score tiles and the
// top-kappa rows); same arguments as launch_scores + launch_topk
cudaError_t launch_scores_topk(int d, int64_t batch, int64_t hq, int64_t hkv, int64_t nq, int64_t nk,
                               const double *q_mean, const double *q_var, const double *k_mean, const double *k_var,
                               int comp, double beta, double *logits, int64_t kappa, double top_p, int32_t *kv_index,
                               int32_t *kv_count, uint8_t *mask, double *prob, double *tau, cudaStream_t st, int *launches);
// top_p > 0: cumulative-mass budget (reading A23), kappa = the cap and the kv_index row stride
cudaError_t launch_topk(int64_t rows, int64_t nk, int64_t kappa, double top_p, const double *logits,
                        int32_t *kv_index, int32_t *kv_count, uint8_t *mask, double *prob,
                        double *tau, cudaStream_t st);

// ---------------------------------------------------------------- attention
constexpr int kMaxPeers = 8;
struct AttnArgs {
  int dtype;          // 0 bf16, 1 fp32
  int d;              // head dim
  int B;              // block size
  int64_t batch, hq, hkv, lq, lk, nq, nk;
  const void *q, *k, *v;       // (sorted) inputs
  int64_t qs[3], ks[3], vs[3]; // element strides (batch, head, token)
  const int32_t *kv_index;     // [b, hq, nq, kv_stride] or nullptr = all blocks
  const int32_t *kv_count;     // [b, hq, nq] or nullptr = kappa
  int64_t kv_stride;           // row stride of kv_index (== kappa)
  const int32_t *perm_q;       // [b, hq, lq] or nullptr = identity
  void *out;
  int64_t os[3];
  float *lse;                  // [b, hq, lq] or nullptr
  float scale;
  int dbg_flags;               // profiling-only knobs (0 in normal use)
  // zero-copy (NEXT-2): q/k/v are the ORIGINAL tensors (dense across batch and head:
  // s1 == L*s2, s0 == H*s1) and rows are fetched through pi_q / pi_k with TMA
  // tile::gather4 (4 rows per instruction) instead of reading permuted copies
  int gather;
  const int32_t *perm_k;       // [b, hkv, lk] (gather only)
  // fused output collective (head-parallel all-gather over NVLink peer memory): when
  // n_peers > 0 every output row is stored to each out_peers[p] (same offsets / strides
  // as out) instead of out — the peers' symmetric buffers, pre-offset to this rank's heads
  int n_peers;
  void *out_peers[kMaxPeers];
  // NVLS multicast (ba_sparse_attn_multicast): when set, every output row is stored once
  // with multimem.st to this multicast address (same offsets / strides as out)
  void *out_mc;
  // device-detected errors (two mapped host words, or nullptr): word kErrEmptyRow is
  // set when a query block's kv_count < 1 (its rows get O = 0, LSE = -inf), word
  // kErrBadIndex when a kv_index entry is outside [0, N_k) (the entry is skipped).
  // One word per error with plain idempotent stores: no read-modify-write, so no
  // system-scope atomics over PCIe are needed.
  unsigned int *err_flag;
  // set by the pair kernel's launcher (NEXT-2): O is dense [b, hq, lq, d] bf16 and goes to `out`
  // (no peers / multicast), so full 128-row blocks are staged in shared memory and written to
  // their rows pi_q(i) by TMA tile::scatter4 (4 rows per instruction) instead of per-thread stores
  int scatter;
};
constexpr int kErrEmptyRow = 0, kErrBadIndex = 1;
BA_HOST_DEVICE_INLINE void flag_error(unsigned int *f, int which) {
  if (f) reinterpret_cast<volatile unsigned int *>(f)[which] = 1u;
}
cudaError_t launch_attn_simt(const AttnArgs &a, cudaStream_t st);
cudaError_t launch_attn_sm100(const AttnArgs &a, cudaStream_t st);
bool attn_sm100_supported(const AttnArgs &a);
bool attn_sm100_dual64();
cudaError_t launch_attn_pp(const AttnArgs &a, cudaStream_t st);
bool attn_pp_supported(const AttnArgs &a);
cudaError_t launch_attn_pp2(const AttnArgs &a, cudaStream_t st);
bool attn_pp2_supported(const AttnArgs &a);

// ---------------------------------------------------------------- NEXT-3: oracle block mass
struct MassArgs {
  int d, B;
  int64_t batch, hq, hkv, lq, lk, nq, nk;
  const void *q, *k;            // Q', K' (sorted copies), bf16
  int64_t qs[3], ks[3];
  const float *lse;             // [b, hq, lq] natural-log row LSE of the dense softmax, sorted order
  float scale;
  const int32_t *kv_index;      // selection for the captured mass (or nullptr)
  const int32_t *kv_count;
  int64_t kv_stride;
  float *m_hat;                 // [b, hq, nq, nk] or nullptr (no mass pass)
  float *captured;              // [b, hq, nq] or nullptr
  float *s_max, *s_min;         // [b, hq, nq, nk] token-logit extremes S = Q'.K' (unscaled), or nullptr
};
bool block_mass_supported(const MassArgs &a);
cudaError_t launch_block_mass(const MassArgs &a, cudaStream_t st);
// Eq. logits-bound: per-block radius R and max norm M (fp64) of a sorted copy
cudaError_t launch_block_radius(int dtype, int d, const void *x, int64_t batch_heads, int64_t L, int B,
                                const double *mean, double *R, double *M, cudaStream_t st);
cudaError_t launch_deviation_finalize(int64_t batch, int64_t hq, int64_t hkv, int64_t nq, int64_t nk, const double *rq,
                                      const double *mq, const double *rk, const double *mk, const double *logit,
                                      const float *smax, const float *smin, double inv_sqrt_d, double *U, double *dev,
                                      cudaStream_t st);

}  // namespace baatt

