/*
 * ba_attn.h — C ABI of libbaatt.so, the B200 (sm_100a) hot path of
 * Block Approximate Sparse Attention (BA-Att, arXiv 2605.19726).
 *
 * The ABI follows the paper's statement of the problem, Algorithm 1
 * (PAPER.md P:527-569): REQUIRE Q, K, V; block size B; per-query-block budget
 * kappa; compensation weight beta  ->  RETURN sparse attention
 * outputs in the original token order.
 *
 *   ba_select       Alg. 1 steps 1-10: norm ranking of Q and K
 *                   (s = ||x||_2), permuted copies Q', K', V'
 *                   (P:537), block means / per-dimension variances
 *                   (P:282), block logits
 *                   l = Qbar.Kbar/sqrt(d) (Eq. block-logit), the
 *                   diagonal-variance compensation Delta (Eq.
 *                   diag-variance-form), l' = l + beta*Delta
 *                   (P:553-556), m' = softmax_row(l') and the
 *                   top-kappa block mask M.
 *   ba_sparse_attn  Alg. 1 steps 11-12: non-causal block-sparse
 *                   attention of Q' over the K'/V' blocks with M = 1,
 *                   online softmax renormalised over the selected support
 *                   (P:263-264), rows written back to the original
 *                   order via pi_q^{-1}.
 *   ba_attention    both, end to end.
 *
 * Conventions (all calls):
 *  - Device pointers unless a name says _host.  The library never allocates
 *    or frees memory: the caller owns every buffer and the stream, and the
 *    buffers must stay alive until the stream work completes.  Scratch comes
 *    from a caller-provided workspace (sizes from the *_workspace_size calls).
 *  - All calls are stream-ordered and asynchronous: they enqueue kernels on
 *    `stream` and return without synchronising.  A launch failure is reported
 *    as BA_ERR_CUDA (cudaGetLastError); an asynchronous fault surfaces at the
 *    caller's next synchronisation.
 *  - Validation is synchronous and happens before any launch; on error
 *    nothing is enqueued and ba_last_error() names the offending field.
 *  - No C++ exception crosses the ABI.  The library is thread-safe for
 *    concurrent calls on different streams (no global mutable state other
 *    than idempotent per-device kernel attributes, the thread-local error
 *    string, ba_attention_host's two cached copy streams per device and the
 *    device-error latch of ba_check_errors: 8 bytes of mapped pinned host
 *    memory, allocated once per process).
 *  - Tensor layout: element (b, h, t, c) of q/k/v/out lives at
 *    base + b*stride[0] + h*stride[1] + t*stride[2] + c (element units; the
 *    feature stride is 1).  Strides and base pointers must be 16-byte aligned
 *    (TMA).  d = head_dim is also the value dimension.
 *  - Attention is non-causal (bidirectional) only (diffusion LMs and
 *    DiTs).
 *  - Numerics: bf16 inputs run on tcgen05 tensor cores with fp32
 *    accumulation and fp32 online softmax; fp32 inputs run an fp32 SIMT
 *    path.  Selection (stats, scores, softmax, top-kappa) is computed in fp64
 *    so that masks match the fp64 oracle except at exact-threshold near-ties.
 */
#ifndef BA_ATTN_H_
#define BA_ATTN_H_

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BA_ABI_VERSION 1

typedef enum {
  BA_OK = 0,
  BA_ERR_INVALID_ARGUMENT = 1,   /* NULL pointer, non-positive size, bad enum, density not in (0,1] */
  BA_ERR_SHAPE_MISMATCH = 2,     /* heads_q % heads_kv != 0, misaligned stride / pointer */
  BA_ERR_UNSUPPORTED = 3,        /* valid but not implemented (head_dim, block_size, dtype combo) */
  BA_ERR_WORKSPACE_TOO_SMALL = 4,
  BA_ERR_CUDA = 5,               /* a CUDA runtime call or launch failed */
  BA_ERR_EMPTY_MASK_ROW = 6      /* a query block with kv_count < 1 reached the attention (every mask row
                                    must be non-empty); detected on the device, reported by
                                    ba_check_errors / the next attention call (see below) */
} ba_status;

typedef enum { BA_DTYPE_BF16 = 0, BA_DTYPE_FP32 = 1 } ba_dtype;

/* Which sides are norm-ranked (ablation Table). */
typedef enum { BA_SORT_NONE = 0, BA_SORT_Q = 1, BA_SORT_K = 2, BA_SORT_QK = 3 } ba_sort_mode;

/* Compensation of the block logits: none; the diagonal-variance form
 * Delta = (1/d) sum_t (VarQ_t Kbar_t^2 + VarK_t Qbar_t^2 + VarQ_t VarK_t)
 * (Eq. diag-variance-form), the default; or the exact covariance
 * form Delta = (1/d) tr(SigmaQ SigmaK) with full per-block covariances
 * (Eq. cov-comp; NEXT-4) — O(N d^2) workspace per side and
 * 2 N_q N_k d^2 FLOP per head, for small L and diagnostics. */
typedef enum { BA_COMP_NONE = 0, BA_COMP_DIAG = 1, BA_COMP_EXACT = 2 } ba_comp_mode;

/* Budget rule ("under different computational budgets"; Alg. 1 step 10
 * P:560 top-kappa).
 *   BA_SELECT_TOPK  every query block keeps kappa = round(density*N_k) blocks.
 *   BA_SELECT_TOPP  cumulative mass (reading A23): order a row by
 *                   (-m', g_k) and keep the shortest prefix whose mass reaches
 *                   top_p, at most kappa(density) blocks (density = 1: no cap);
 *                   kv_count[row] = that length, kv_index rows keep the
 *                   capacity kappa(density) as their stride. */
typedef enum { BA_SELECT_TOPK = 0, BA_SELECT_TOPP = 1 } ba_select_mode;

typedef struct {
  int32_t batch;        /* b >= 1 */
  int32_t heads_q;      /* H_q >= 1 */
  int32_t heads_kv;     /* H_kv >= 1, heads_q % heads_kv == 0 (GQA: q-head h uses kv-head h / (H_q/H_kv)) */
  int32_t head_dim;     /* d in {64, 128} */
  int64_t len_q;        /* L_q >= 1; need not be a multiple of block_size (ragged last block) */
  int64_t len_k;        /* L_k >= 1 */
  int32_t block_size;   /* B in {64, 128}: N_q = ceil(L_q/B), N_k = ceil(L_k/B) */
  int32_t dtype;        /* ba_dtype of q, k, v, out */
  int64_t q_stride[3];  /* element strides for (batch, head, token); feature stride is 1 */
  int64_t k_stride[3];
  int64_t v_stride[3];
  int64_t o_stride[3];
} ba_problem;

typedef struct {
  int32_t sort;          /* ba_sort_mode; default BA_SORT_QK */
  int64_t sort_window;   /* 0 = global sort; w > 0 sorts each run of w tokens independently ("(windowed) sort") */
  int32_t comp;          /* ba_comp_mode; default BA_COMP_DIAG */
  float beta;            /* compensation weight; default 1 */
  int32_t select;        /* ba_select_mode; BA_SELECT_TOPK */
  float density;         /* rho in (0, 1]; kappa = max(1, min(N_k, floor(rho*N_k + 1/2))) (reading A2) */
  float top_p;           /* BA_SELECT_TOPP only: in (0, 1] (else BA_ERR_INVALID_ARGUMENT) */
  float softmax_scale;   /* 0 => 1/sqrt(head_dim) (Eq. sdpa) */
} ba_params;

/* Selection produced by ba_select and consumed by ba_sparse_attn /
 * ba_sparse_attn_gather.  Every buffer is caller-allocated device memory.
 * Required fields: perm_q, perm_k, kv_index, kv_count.  q_sorted, k_sorted,
 * v_sorted: required by ba_sparse_attn; NULL = ba_select does not
 * materialise that permuted copy (zero-copy: ba_sparse_attn_gather reads the
 * rows through pi_q / pi_k instead).  Optional (NULL = not written):
 * everything else. */
typedef struct {
  int32_t *perm_q;       /* [b, H_q, L_q]   sorted position -> original token index (pi_q) */
  int32_t *perm_k;       /* [b, H_kv, L_k]  pi_k */
  void *q_sorted;        /* [b, H_q, L_q, d] contiguous, dtype: Q'_i = Q_{pi_q(i)} */
  void *k_sorted;        /* [b, H_kv, L_k, d] contiguous: K'_j = K_{pi_k(j)} */
  void *v_sorted;        /* [b, H_kv, L_k, d] contiguous: V'_j = V_{pi_k(j)} */
  int32_t *kv_index;     /* [b, H_q, N_q, kappa] selected key blocks g_k, strictly ascending */
  int32_t *kv_count;     /* [b, H_q, N_q] number of valid entries per row (== kappa for TOPK, <= kappa for TOPP) */
  uint8_t *mask;         /* [b, H_q, N_q, N_k] M in {0,1} */
  double *block_prob;    /* [b, H_q, N_q, N_k] m' = softmax_row(l') */
  double *logits;        /* [b, H_q, N_q, N_k] l' = l + beta*Delta */
  double *threshold;     /* [b, H_q, N_q] tau = m' of the last (kv_count-th largest) selected block */
  double *q_mean;        /* [b, H_q, N_q, d] Qbar over the sorted blocks */
  double *q_var;         /* [b, H_q, N_q, d] population variance per dimension */
  double *k_mean;        /* [b, H_kv, N_k, d] */
  double *k_var;         /* [b, H_kv, N_k, d] */
  float *q_key;          /* [b, H_q, L_q] sort key fp32(||q||^2) in ORIGINAL order (reading A4) */
  float *k_key;          /* [b, H_kv, L_k] */
} ba_selection;

/* ABI version compiled into the library (== BA_ABI_VERSION of this header). */
int ba_abi_version(void);

/* N_q, N_k and kappa for a problem (no device work).  Returns
 * BA_ERR_INVALID_ARGUMENT / BA_ERR_UNSUPPORTED on a bad problem. */
ba_status ba_selection_sizes(const ba_problem *prob, const ba_params *params,
                             int64_t *kappa, int64_t *n_q, int64_t *n_k);

/* Scratch bytes needed by ba_select (sort buffers, histograms, stats and the
 * fp64 score map when not supplied).  0 on an invalid problem.  ba_select
 * supports N_k <= 28672 key blocks (its top-kappa row buffer lives in shared
 * memory): larger problems return BA_ERR_UNSUPPORTED before any launch. */
size_t ba_select_workspace_size(const ba_problem *prob, const ba_params *params);

/* Scratch bytes needed by ba_attention: ba_select's scratch plus every
 * required ba_selection buffer (they are carved from the workspace). */
size_t ba_attention_workspace_size(const ba_problem *prob, const ba_params *params);

/* Alg. 1 steps 1-10.  q, k, v: device tensors in the ba_problem layout.
 * Writes every non-NULL buffer of *sel.  workspace: >= ba_select_workspace_size
 * bytes, 256-byte aligned. */
ba_status ba_select(const ba_problem *prob, const ba_params *params,
                    const void *q, const void *k, const void *v,
                    const ba_selection *sel, void *workspace, size_t workspace_bytes,
                    cudaStream_t stream);

/* Alg. 1 steps 11-12.  Reads sel->q_sorted, k_sorted, v_sorted, kv_index,
 * kv_count, perm_q (a caller may inject its own selection: kv_index rows must
 * be ascending, unique, in [0, N_k), with kv_count >= 1).  out: original
 * token order, ba_problem o_stride layout.  lse: optional [b, H_q, L_q] fp32
 * natural-log log-sum-exp of the scaled logits per query row, original order.
 *
 * Injected selections are checked ON THE DEVICE (checking them on the host
 * would need a synchronising copy): a query block whose kv_count < 1 violates
 * the non-empty-row precondition — its rows are written as O = 0,
 * LSE = -inf (deterministic, never unwritten accumulator memory) and
 * BA_ERR_EMPTY_MASK_ROW is latched; a kv_index entry outside [0, N_k) is
 * skipped and BA_ERR_INVALID_ARGUMENT latched.  A latched error is returned
 * (and cleared) by ba_check_errors, or by the next ba_sparse_attn* /
 * ba_attention / ba_dense_attn call on any thread once the faulting kernel
 * has finished — like CUDA's asynchronous errors.  The latch is one pair of
 * words of mapped pinned host memory per process, allocated on first use.
 *
 * bf16 with head_dim 128 always runs a tcgen05 kernel; problems those
 * kernels cannot take (N_k > 32768 key blocks) return BA_ERR_UNSUPPORTED —
 * never a silent SIMT fallback.  bf16 head_dim 64 and every fp32 problem run
 * the SIMT kernel (ba_attention_kernel_name says which). */
ba_status ba_sparse_attn(const ba_problem *prob, const ba_params *params,
                         const ba_selection *sel, void *out, float *lse,
                         cudaStream_t stream);

/* Alg. 1 steps 11-12 reading the ORIGINAL tensors through the permutations
 * (NEXT-2, zero-copy): Q'_i = Q_{pi_q(i)} is always read in place, and
 * K'_j = K_{pi_k(j)}, V'_j = V_{pi_k(j)} too when sel->k_sorted /
 * v_sorted are NULL (else those copies are read) — the attention kernels fetch
 * 4 token rows per TMA tile::gather4 instruction through perm_q / perm_k, so
 * ba_select need not write the corresponding copies.  q, k, v: the tensors
 * passed to ba_select.  Reads sel->perm_q, perm_k, kv_index, kv_count.
 * Requirements (else BA_ERR_UNSUPPORTED, nothing enqueued): bf16,
 * head_dim 128, the gathered tensors dense across (batch, head)
 * (stride[1] == L*stride[2], stride[0] == H*stride[1]), b*H*L < 2^31; B = 64
 * uses the dual-tile kernel; not with BA_ATTN_K5=2cta.  Performance: gathering
 * K/V costs ~2.3x attention time on B200, gathering Q is free. */
ba_status ba_sparse_attn_gather(const ba_problem *prob, const ba_params *params,
                                const void *q, const void *k, const void *v,
                                const ba_selection *sel, void *out, float *lse,
                                cudaStream_t stream);

/* What ba_sparse_attn_gather supports for this problem: 3 = Q, K and V read
 * through the permutations (no copies at all), 1 = Q only (K'/V' copies
 * needed), 0 = neither (use ba_sparse_attn).  No device work. */
int ba_zero_copy_supported(const ba_problem *prob, const ba_params *params);

/* Alg. 1 steps 11-12 with the head-parallel output collective fused into the
 * epilogue: every output row is stored to EACH of the
 * n_peers buffers out_peers[0..n_peers) (device pointers valid in this
 * process — e.g. the peers' symmetric-memory buffers mapped over NVLink /
 * NVSwitch, each pre-offset to this rank's head slice; same o_stride layout),
 * so after a barrier every rank holds the whole O without an all-gather pass.
 * Otherwise as ba_sparse_attn (reads the permuted copies).  1 <= n_peers <= 8;
 * bf16, head_dim 128 (the tcgen05 pair / single-CTA kernels), else
 * BA_ERR_UNSUPPORTED.  The library performs no cross-rank synchronisation: the
 * caller orders the peers' reads after every rank's kernel (e.g. a symmetric
 * memory barrier). */
ba_status ba_sparse_attn_peers(const ba_problem *prob, const ba_params *params,
                               const ba_selection *sel, void *const *out_peers, int n_peers,
                               float *lse, cudaStream_t stream);

/* As ba_sparse_attn_peers, but every output row is stored ONCE, with multimem.st
 * (NVLS, NVLink SHARP), to out_multicast: a multicast device address (e.g. torch
 * symmetric memory's multicast_ptr) pre-offset to this rank's head slice, so the
 * NVSwitch replicates each store into every rank's copy — one store instruction
 * and one NVLink egress per row instead of n_peers unicast stores.  Same layout
 * rules as ba_sparse_attn_peers; bf16, head_dim 128 (tcgen05 kernels), else
 * BA_ERR_UNSUPPORTED.  The caller orders the peers' reads after every rank's
 * kernel (a symmetric-memory barrier). */
ba_status ba_sparse_attn_multicast(const ba_problem *prob, const ba_params *params,
                                   const ba_selection *sel, void *out_multicast, float *lse,
                                   cudaStream_t stream);

/* Alg. 1 steps 11-12 for a contiguous range of WORK UNITS only —
 * the uneven multi-GPU split of SURVEY §8(e) (e.g. 28 heads over 8 GPUs):
 * unit u = (b*H_q + h)*N_q + g_q is query block g_q of head h of batch b, and
 * every row of the units in [unit_begin, unit_end) is computed as
 * ba_sparse_attn computes it and stored at its ORIGINAL token position in
 * each of out[0..n_out); rows of other units are not written.  Bit-identical
 * to ba_sparse_attn when both range ends fall on an even query block or a
 * head boundary: the B = 64 dual-tile kernel pairs query blocks (2p, 2p+1)
 * and groups key blocks by the pair's union, so a block's rounding depends
 * on its partner (the B = 128 kernels' rows depend only on their own list);
 * otherwise equal within the parity tolerance.  Every (b, h) problem
 * is independent (Alg. 1 is per head), so rank r of G can run units
 * [r*U/G, (r+1)*U/G) after a ba_select over the heads it touches.  n_out = 1:
 * plain stores (any kernel); 1 < n_out <= 8: peer stores as
 * ba_sparse_attn_peers (same kernel requirements; the caller synchronises the
 * peers).  Reads the permuted copies, kv_index, kv_count, perm_q.  lse as
 * ba_sparse_attn (only the units' rows written).  Launches one kernel per run
 * of whole GQA groups and one per partial head.  Errors: range outside
 * [0, b*H_q*N_q) or n_out outside 1..8 -> BA_ERR_INVALID_ARGUMENT; an empty
 * range enqueues nothing and returns BA_OK. */
ba_status ba_sparse_attn_units(const ba_problem *prob, const ba_params *params,
                               const ba_selection *sel, int64_t unit_begin, int64_t unit_end,
                               void *const *out, int n_out, float *lse, cudaStream_t stream);

/* ba_select + attention with the selection carved from the workspace
 * (>= ba_attention_workspace_size bytes), on the permuted copies
 * (ba_sparse_attn) — the faster path on B200.  The environment
 * variable BA_ZERO_COPY=1 runs ba_sparse_attn_gather with no copies, =2 with
 * only Q read in place, when ba_zero_copy_supported allows it. */
ba_status ba_attention(const ba_problem *prob, const ba_params *params,
                       const void *q, const void *k, const void *v,
                       void *out, float *lse, void *workspace, size_t workspace_bytes,
                       cudaStream_t stream);

/* Dense (all N_k blocks, no ranking) attention through the same tensor-core
 * kernel: the 1/rho speed-of-light reference for the sparse path.  Same
 * layouts as ba_attention; no workspace. */
ba_status ba_dense_attn(const ba_problem *prob, const ba_params *params,
                        const void *q, const void *k, const void *v,
                        void *out, float *lse, cudaStream_t stream);

/* End-to-end from HOST memory: copies q, k, v (host, contiguous [b,H,L,d];
 * pinned for asynchronous copies) into device staging carved from the
 * workspace, runs ba_attention, copies the output back to out_host
 * (contiguous [b,H_q,L_q,d]).  Stream-ordered: synchronise `stream` before
 * reading out_host.  Strides in *prob are ignored (contiguous assumed). */
size_t ba_attention_host_workspace_size(const ba_problem *prob, const ba_params *params);
ba_status ba_attention_host(const ba_problem *prob, const ba_params *params,
                            const void *q_host, const void *k_host, const void *v_host,
                            void *out_host, void *workspace, size_t workspace_bytes,
                            cudaStream_t stream);

/* NEXT-3 fidelity diagnostic: the oracle block distribution (Eq. oracle-dist,
 * P:300-312) m_hat[g_q, g_k] = (1/|I(g_q)|) sum_{i in I(g_q)} sum_{j in J(g_k)}
 * A_ij of the DENSE softmax A = softmax(Q' K'^T * scale) in the norm-sorted
 * block space, and the selection's captured mass
 * captured[g_q] = sum over the selected g_k of m_hat[g_q, g_k].
 * Reads sel->q_sorted, k_sorted, v_sorted (and kv_index / kv_count when
 * captured != NULL).  m_hat: [b, H_q, N_q, N_k] fp32; captured: [b, H_q, N_q]
 * fp32 or NULL.  Runs a dense pass (for the row log-sum-exp) and a second
 * S = Q'K'^T pass on the tensor cores.  bf16, head_dim 128, block_size 128
 * (else BA_ERR_UNSUPPORTED).  workspace >= ba_block_mass_workspace_size. */
size_t ba_block_mass_workspace_size(const ba_problem *prob, const ba_params *params);
ba_status ba_block_mass(const ba_problem *prob, const ba_params *params, const ba_selection *sel,
                        float *m_hat, float *captured, void *workspace, size_t workspace_bytes,
                        cudaStream_t stream);

/* NEXT-3 fidelity diagnostic: the bound of Eq. logits-bound
 *   U[g_q, g_k] = (R^Q M^K + M^Q R^K + R^Q R^K) / sqrt(d),
 *   R = max_{i in block} ||x_i - xbar||_2, M = max_{i in block} ||x_i||_2,
 * and the observed maximum logit deviation it bounds (Fig. 2, P:386-392;
 * Eq. logit-deviation)
 *   max_dev[g_q, g_k] = max_{i in I(g_q), j in J(g_k)} |Q'_i.K'_j/sqrt(d) - Qbar.Kbar/sqrt(d)|
 * per block pair of the norm-sorted block space of a selection (the paper's
 * "red group").  Reads sel->q_sorted, k_sorted and the fp64 block means
 * sel->q_mean, k_mean (pass those buffers to ba_select).  bound_u, max_dev:
 * [b, H_q, N_q, N_k] fp64 (either may be NULL).  R and M are fp64 against the
 * fp64 means; the token logits come from a dense S = Q'K'^T pass on the
 * tensor cores (bf16 inputs, fp32 accumulation: |error| <= d*2^-24 * M^Q M^K),
 * the block logit from an fp64 DMMA.  bf16, head_dim 128, block_size 128
 * (else BA_ERR_UNSUPPORTED).  workspace >= ba_deviation_workspace_size. */
size_t ba_deviation_workspace_size(const ba_problem *prob, const ba_params *params);
ba_status ba_deviation(const ba_problem *prob, const ba_params *params, const ba_selection *sel,
                       double *bound_u, double *max_dev, void *workspace, size_t workspace_bytes,
                       cudaStream_t stream);

/* Name of the attention kernel ba_sparse_attn / ba_attention / ba_dense_attn
 * run for this problem: "attn_sm100_tcgen05" (bf16, d = 128, B in {64, 128}:
 * tcgen05 tensor cores, TMA, TMEM; B = 64 pairs two query blocks per 128-row
 * tile) or "attn_simt" (fp32 inputs, and bf16 d = 64).  "" on an invalid
 * problem. */
const char *ba_attention_kernel_name(const ba_problem *prob, const ba_params *params);

/* Synchronises `stream`, then returns (and clears) an error the attention
 * kernels latched on the device (BA_ERR_EMPTY_MASK_ROW: a query block with
 * kv_count < 1; BA_ERR_INVALID_ARGUMENT: a kv_index entry outside
 * [0, N_k)), or BA_ERR_CUDA if the synchronisation failed; BA_OK otherwise. */
ba_status ba_check_errors(cudaStream_t stream);

/* Number of kernel launches the last successful call on this thread enqueued. */
int ba_last_launch_count(void);

const char *ba_status_string(ba_status status);
/* Thread-local detail of the last error on this thread ("" if none). */
const char *ba_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* BA_ATTN_H_ */
