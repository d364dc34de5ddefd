/*
 * qrita_b200.h — C ABI of the B200-native exact Top-k / Top-p truncation library
 * (libqrita_b200.so).  Plain pointers and sizes only; no torch or C++ types.
 *
 * Every entry point replaces one piece of the reference operator surface
 * (paths relative to the reference tree, arxiv/paper_2602_01518):
 *
 *   qrita_topk_topp          <- pkg/src/sigmatop/engine.py:82-113   run_batch (per-row loop over
 *                               pkg/src/sigmatop/pipeline.py:199-239 truncate_topk_topp, which
 *                               itself dispatches to truncate_topk :140-158 / truncate_topp :161-196)
 *                               and the paper's GPU operator shape
 *                               _topk_topp_triton_kernel(LOGITS, BUFFER, OUTPUT, ..., K, P, ..., INPLACE)
 *                               (PAPER.md:176-188): per-row K/P, [B,V] logits, caller scratch, in-place.
 *   qrita_workspace_bytes    <- the paper's caller-provided BUFFER[num_programs, V]
 *   qrita_get_status         <- pkg/src/sigmatop/core.py:120-140 validate_batch (non-finite logits,
 *                               k out of [1,V], p out of (0,1]) as raised by engine.py:76-79
 *   qrita_strerror           <- the ValueError texts of core.py:126-139 / pipeline.py:148-149,168-169
 *
 * Semantics (bit-exact against pkg/src/sigmatop/oracle.py:70-89): per row, keep the first k entries of
 * the stable descending order (value desc, index asc, -0.0 == +0.0); renormalise the fp64 softmax over
 * those survivors with the full-row max; keep the shortest prefix whose exactly-rounded probability sum
 * reaches p.  k == V disables top-k, p == 1 disables top-p.  Kept entries are written bit-identical to
 * the input, removed entries become -inf, in the input dtype.
 *
 * All pointers are DEVICE pointers unless stated; every call is stream-ordered and never synchronises
 * except qrita_get_status.  The library keeps no global state besides constant tables; the caller owns
 * every buffer.  Calls on different streams must use different workspaces.
 */
#ifndef QRITA_B200_H
#define QRITA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* cudaStream_t without pulling in the CUDA headers. */
typedef struct CUstream_st *qrita_stream_t;

/* input / output dtypes */
enum {
  QRITA_DTYPE_F32 = 0,
  QRITA_DTYPE_BF16 = 1
};

/* flags — the reference EngineConfig ablation switches (engine.py:26-40) plus in-place */
enum {
  QRITA_SEARCH_BINARY   = 1 << 0, /* 1 pivot per pass instead of 3 (pivot_search.py:136-140, 241-244) */
  QRITA_NO_SIGMA        = 1 << 1, /* sigma_trunc_enabled=False: never gather outliers                */
  QRITA_FORCE_FALLBACK  = 1 << 2, /* force_fallback=True: gather, but search the full row           */
  QRITA_NO_DUP          = 1 << 3, /* duplication_handling_enabled=False: keep whole boundary cluster*/
  QRITA_INPLACE         = 1 << 4, /* out == logits (pipeline.py:72-74)                               */
  QRITA_RESERVED_5      = 1 << 5, /* reserved (rejected)                                            */
  QRITA_DEBUG_TIMING    = 1 << 6, /* record per-row tail phase timestamps (qrita_get_timing)        */
  QRITA_STAGED          = 1 << 7, /* force the staged 3-kernel pipeline (prep / stream / tail) even
                                     when the fused single-kernel path applies                      */
  QRITA_TP_NO_TOPP_ROWS = 1 << 8  /* vocab-sharded call only: the caller guarantees no row is top-p
                                     only (k == V_global, p < 1), so the top-p rounds are skipped   */
};

/* return codes */
enum {
  QRITA_OK = 0,
  QRITA_EINVAL_ARG = 1,   /* bad shape / pointer / flag combination        */
  QRITA_EINVAL_K = 2,     /* some row has k outside [1, V]                  */
  QRITA_EINVAL_P = 3,     /* some row has p outside (0, 1]                  */
  QRITA_ENONFINITE = 4,   /* some logit is NaN or +-inf                     */
  QRITA_EWORKSPACE = 5,   /* workspace too small / misaligned              */
  QRITA_ECUDA = 6,        /* a CUDA runtime call failed                     */
  QRITA_ENCCL = 7         /* a collective of the vocab-sharded variant failed */
};

/* Per-row accounting, field-for-field the reference RowMetrics (core.py:72-81) plus kept_count
 * (TruncationOutput.kept_count, core.py:84-90) and which physical path ran. */
typedef struct qrita_row_metrics {
  int32_t trunc_hit;         /* sigma pre-filter hit (reference rule: count > k, or mass > p) */
  int32_t outlier_count;     /* entries strictly above the sigma threshold                    */
  double  outlier_prob_sum;  /* top-p-only rows: softmax mass of the outliers                 */
  int32_t k_search_iters;    /* pivot passes of the top-k search                              */
  int32_t p_search_iters;    /* pivot passes of the top-p search                              */
  int32_t fallback_used;     /* reference semantics: not trunc_hit                            */
  int32_t kept_count;        /* number of kept entries                                        */
  int32_t full_row_path;     /* 1 if this build searched the full row (miss / capacity)       */
  int32_t row_passes;        /* passes over the row's logits: 1 = the single streaming pass; each   */
                             /* full-row re-read of a fallback / full-row path adds one           */
} qrita_row_metrics;

/* Bytes of device workspace needed for a [B, V] call.  The workspace must be zeroed once before its
 * first use (qrita_workspace_init); afterwards every call leaves it clean for the next one. */
size_t qrita_workspace_bytes(int B, int V, int dtype, int flags);

/* cudaMemsetAsync(ws, 0, bytes, stream). */
int qrita_workspace_init(void *workspace, size_t ws_bytes, qrita_stream_t stream);

/*
 * Exact Top-k + Top-p truncation of a [B, V] row-major logit matrix.
 *   logits      device [B, ld_in] f32 or bf16 (dtype); rows are the first V columns
 *   k           device int64 [B]   (1 <= k <= V; k == V disables top-k)
 *   p           device float64 [B] (0 < p <= 1;  p == 1 disables top-p) — fp64, as core.py:63
 *   out         device [B, ld_out] same dtype; may equal logits iff flags & QRITA_INPLACE
 *   kept_count  device int32 [B] or NULL
 *   metrics     device qrita_row_metrics [B] or NULL
 *   sample_size prefix length of the sigma statistics (sigma_trunc.py:69-82; default 4096)
 * Invalid k / p / non-finite rows are reported through qrita_get_status; their output is undefined.
 */
int qrita_topk_topp(const void *logits, int64_t ld_in, int dtype, int B, int V,
                    const int64_t *k, const double *p,
                    void *out, int64_t ld_out,
                    int32_t *kept_count, qrita_row_metrics *metrics,
                    void *workspace, size_t ws_bytes, int flags, int sample_size,
                    qrita_stream_t stream);

/* qrita_topk_topp plus the kept-column list (SURVEY.md 8b kept_idx): kept_idx DEVICE int32 [B, ld_idx]
 * (ld_idx >= V) receives each row's kept column indices in unspecified order, kept_count[row] of them
 * (kept_count or metrics must be given).  out may be NULL: index-only output, no masked logits are
 * written (V * sizeof(dtype) read + kept * 4 written per row).  Same validation and status as
 * qrita_topk_topp; QRITA_INPLACE requires out. */
int qrita_topk_topp_idx(const void *logits, int64_t ld_in, int dtype, int B, int V,
                        const int64_t *k, const double *p,
                        void *out, int64_t ld_out,
                        int32_t *kept_idx, int64_t ld_idx,
                        int32_t *kept_count, qrita_row_metrics *metrics,
                        void *workspace, size_t ws_bytes, int flags, int sample_size,
                        qrita_stream_t stream);

/* Same as qrita_topk_topp, for profiling: records `prep_done_event` after the preparation kernel and
 * `stream_done_event` after the streaming kernel (cudaEvent_t each, may be NULL).  A non-NULL event
 * serialises the launches around it (no programmatic overlap), so each kernel can be timed alone
 * with events (bench.py's roofline measurement). */
int qrita_topk_topp_ex(const void *logits, int64_t ld_in, int dtype, int B, int V,
                       const int64_t *k, const double *p,
                       void *out, int64_t ld_out,
                       int32_t *kept_count, qrita_row_metrics *metrics,
                       void *workspace, size_t ws_bytes, int flags, int sample_size,
                       qrita_stream_t stream, void *prep_done_event, void *stream_done_event);

/*
 * Host-buffer variant (the reference's run_batch takes host arrays, engine.py:82-113): logits / out
 * are HOST [B, V] row-major arrays, k / p are HOST arrays.  Page-locked buffers are copied by DMA
 * directly; pageable buffers are staged through two library-owned page-locked slots per direction,
 * filled / drained by a pool of host threads (QRITA_HOST_COPY_THREADS) one chunk ahead of / behind
 * the DMA — with a pageable `out_host` the call returns only once the result is in it.  Row chunks of `chunk_rows` rows are copied in, truncated and copied back on three
 * streams owned by the library (upload / truncate / download), ordered by per-chunk events, so both
 * PCIe directions and the kernels overlap.  `scratch` is a DEVICE buffer of
 * qrita_host_scratch_bytes(B, V, dtype, chunk_rows) bytes, 256-byte aligned (no initialisation
 * needed).  The work is ordered after everything already enqueued on `stream`, and `stream` waits
 * for all of it: synchronise `stream` before reading `out`.  kept_count / metrics: DEVICE or NULL.
 * Invalid rows are reported by qrita_get_status_host.
 * Sparse downloads: when every row has 1 <= k < V, k <= 4096 (top-k active) — and unless a pageable
 * logits_host meets a page-locked out_host — the kernels write each row's kept columns instead of its
 * masked row, only those (and the counts) cross PCIe, and host threads build the masked rows from
 * logits_host (-inf fill, kept entries copied: bit-identical); the call then returns with out_host
 * complete.  qrita_host_download_bytes(B, V, dtype, k_host, logits_host, out_host) gives the bytes a
 * call downloads (QRITA_HOST_DENSE=1 / QRITA_HOST_SPARSE=1 force either form).
 */
size_t qrita_host_scratch_bytes(int B, int V, int dtype, int chunk_rows);
int64_t qrita_host_download_bytes(int B, int V, int dtype, const int64_t *k_host, const void *logits_host,
                                  const void *out_host);
int qrita_topk_topp_host(const void *logits_host, int dtype, int B, int V,
                         const int64_t *k_host, const double *p_host, void *out_host,
                         int32_t *kept_count, qrita_row_metrics *metrics,
                         void *scratch, size_t scratch_bytes, int chunk_rows, int flags, int sample_size,
                         qrita_stream_t stream);
/* qrita_get_status for the last qrita_topk_topp_host call on `scratch` (same B, V, chunk_rows). */
int qrita_get_status_host(const void *scratch, int B, int V, int dtype, int chunk_rows, int *row, int *col,
                          qrita_stream_t stream);

/*
 * Vocab-sharded (tensor-parallel LM-head) variant — BASELINE cfg5, SURVEY.md 8(b)/8(e).
 *
 * Every rank holds the columns [vocab_offset, vocab_offset + V_shard) of the [B, V_global] logits
 * (shards contiguous, offsets increasing with rank) and receives its shard of the UNSHARDED answer,
 * bit-exact.  Only per-row partials cross ranks (include: what is exchanged, bytes per row):
 *   1. local top-min(k, V_shard) candidates (top-p-only rows: the local max), one all-gather of
 *      (order key, global column) pairs, each rank's list sorted by (value desc, column asc):
 *      <= 8 * k_cap bytes per row per rank; every rank merges the lists into the global top-k and
 *      resolves top-p over it (global stable order, full-row max and survivor normaliser all live
 *      in that set);
 *   2. top-p-only rows only: the exact normaliser (fixed-point limbs, integer all-reduce SUM: exact
 *      and order-independent), then 4 (bf16) / 8 (fp32) radix passes, each an all-reduce SUM of 16
 *      (count, exact mass) partials per row, then one all-reduce of the per-rank boundary-tie counts
 *      (ties are kept in global index order, i.e. rank order).
 *
 *   logits / out   device [B, ld_in] / [B, ld_out] shard (out may equal logits with QRITA_INPLACE)
 *   k, p           device int64 / float64 [B], the GLOBAL targets (k == V_global disables top-k)
 *   k_cap          >= every k < V_global in the batch (rows violating it report QRITA_EINVAL_ARG
 *                  through qrita_get_status); bounds the candidate exchange
 *   kept_count     device int32 [B] or NULL: entries kept in THIS shard
 *   flags          0, QRITA_INPLACE, QRITA_TP_NO_TOPP_ROWS
 *   workspace      qrita_tp_workspace_bytes(...) bytes, zeroed before first use (qrita_workspace_init)
 * Status (non-finite logits of this shard, bad k / p) is read with qrita_get_status(workspace, B).
 */
typedef struct qrita_comm {
  /* in-place all-reduce SUM of `count` unsigned integers of `elem_bytes` (4 or 8) bytes each in the
   * DEVICE buffer `buf`, ordered on `stream`; returns 0 on success */
  int (*all_reduce_sum)(void *buf, size_t count, int elem_bytes, qrita_stream_t stream, void *ctx);
  /* all-gather: DEVICE `send` (bytes_per_rank bytes) of every rank into DEVICE `recv`
   * (world * bytes_per_rank, rank order), ordered on `stream`; returns 0 on success */
  int (*all_gather)(const void *send, void *recv, size_t bytes_per_rank, qrita_stream_t stream, void *ctx);
  void *ctx;
} qrita_comm;

size_t qrita_tp_workspace_bytes(int B, int V_shard, int dtype, int world, int k_cap);

int qrita_topk_topp_tp_comm(const void *logits, int64_t ld_in, int dtype, int B, int V_shard,
                            int V_global, int64_t vocab_offset, const int64_t *k, const double *p,
                            int k_cap, void *out, int64_t ld_out, int32_t *kept_count,
                            void *workspace, size_t ws_bytes, int flags, int rank, int world,
                            const qrita_comm *comm, qrita_stream_t stream);

/* The same over an NCCL communicator (ncclComm_t; NCCL is loaded at run time: libnccl.so.2). */
int qrita_topk_topp_tp(const void *logits, int64_t ld_in, int dtype, int B, int V_shard,
                       int V_global, int64_t vocab_offset, const int64_t *k, const double *p,
                       int k_cap, void *out, int64_t ld_out, int32_t *kept_count,
                       void *workspace, size_t ws_bytes, int flags, int rank, int world,
                       void *nccl_comm, qrita_stream_t stream);

/* NCCL communicator helpers (a library-owned communicator over the ranks of a job): rank 0 creates
 * the 128-byte unique id, the job broadcasts it, every rank calls qrita_nccl_comm_init on its own
 * device.  Return QRITA_OK or QRITA_ENCCL. */
int qrita_nccl_unique_id(void *id_out /* 128 bytes */);
int qrita_nccl_comm_init(void **comm_out, int world, const void *id, int rank);
int qrita_nccl_comm_destroy(void *comm);

/* cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, stream) + stream synchronise (host-staged
 * exchanges of a qrita_comm implemented outside CUDA, e.g. over gloo). */
int qrita_copy_sync(void *dst, const void *src, size_t bytes, qrita_stream_t stream);

/* The reference's sigma_trunc primitives (pkg/src/sigmatop/sigma_trunc.py):
 *   qrita_sigma_table  <- TOPK_TABLE / TOPP_TABLE (tables.py:13-57): copies the 200 embedded entries
 *                         of kind 0 (top-k) or 1 (top-p) into HOST out[n >= 200]; no CUDA call.
 *   qrita_row_stats    <- row_stats (sigma_trunc.py:69-82): DEVICE out[B][2] = (mu, sigma) of the
 *                         first min(sample_size, V) entries of every row, numpy's pairwise sums bit
 *                         for bit; stream-ordered. */
int qrita_sigma_table(int kind, double *out, int n);
int qrita_row_stats(const void *logits, int64_t ld, int dtype, int B, int V, int sample_size, double *out,
                    qrita_stream_t stream);

/* LM-head producer fusion (the reference has no code for this producer — its
 * consumer is truncate_topk_topp, pipeline.py:199-239, ground truth oracle.py:70-89):
 *   logits[b][v] = sum_k hidden[b][k] * weight[v][k]  — hidden [B, d] and weight [V, d] bf16 row-major
 *   (leading dimensions ld_h / ld_w elements, 16-byte aligned), d % 64 == 0, fp32 accumulation on the
 *   tensor cores (tcgen05.mma, TMA-fed), logits fp32 [B, ld_logits].
 *   qrita_lmhead_logits      the plain GEMM (also the reference the fused call is checked against).
 *   qrita_lmhead_topk_topp   the GEMM with the truncation's streaming pass in its epilogue: writes the
 *                            logits once and the exact Top-k/Top-p kept columns (kept_idx [B][ld_idx],
 *                            unordered) and counts — identical to qrita_topk_topp_idx on those logits;
 *                            on a sigma hit the logits are never read back.  Workspace:
 *                            qrita_lmhead_workspace_bytes(B, V); status via qrita_get_status(workspace). */
int qrita_lmhead_logits(const void *hidden, int64_t ld_h, const void *weight, int64_t ld_w, int B, int V, int d,
                        float *logits, int64_t ld_logits, qrita_stream_t stream);
size_t qrita_lmhead_workspace_bytes(int B, int V);
int qrita_lmhead_topk_topp(const void *hidden, int64_t ld_h, const void *weight, int64_t ld_w, int B, int V, int d,
                           const int64_t *k, const double *p, float *logits, int64_t ld_logits, int32_t *kept_idx,
                           int64_t ld_idx, int32_t *kept_count, qrita_row_metrics *metrics, void *workspace,
                           size_t ws_bytes, int flags, qrita_stream_t stream);

/* Synchronises `stream`, then reports the first failing row of the last call on this workspace:
 * returns QRITA_OK or QRITA_EINVAL_K / QRITA_EINVAL_P / QRITA_ENONFINITE, and fills *row / *col
 * (col = first non-finite column, or -1). */
int qrita_get_status(const void *workspace, int B, int *row, int *col, qrita_stream_t stream);

/* Synchronises `stream` and copies the [B][16] tail phase timestamps (ns, %globaltimer) of the last
 * QRITA_DEBUG_TIMING call on this workspace into host memory `out`. */
int qrita_get_timing(const void *workspace, int B, unsigned long long *out, qrita_stream_t stream);

const char *qrita_strerror(int code);

/* Library version, MAJOR*10000 + MINOR*100 + PATCH. */
int qrita_version(void);

#ifdef __cplusplus
}
#endif

#endif /* QRITA_B200_H */
