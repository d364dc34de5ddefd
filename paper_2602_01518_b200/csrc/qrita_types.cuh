// qrita_types.cuh — constants, workspace records and launch parameters shared by the kernels
// and the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "qrita_device.cuh"
#include "qrita_b200.h"

namespace qrita {


// ------------------------------------------------------------------------------------------------
// Constants
// ------------------------------------------------------------------------------------------------
constexpr int kTableSize = 200;  // tables.py:11
constexpr int kChunk = 1024;     // elements per streaming work item (one warp)
constexpr int kCapChunk = 256;   // outliers per chunk staged in shared memory by the streaming warp
constexpr int kCapX = 8192;      // outliers per row: row buffer in HBM and shared-memory staging
constexpr int kSpecTail = 16;    // outliers per tail thread loaded before the row count is known
constexpr int kCapS = 1024;      // top-k survivors whose probabilities are cached in shared memory
constexpr int kCapA = 1024;      // active set of the top-p pivot search (3x as many keys for top-k)
constexpr int kStreamThreads = 256;
constexpr int kMaxTailChunks = 2048;  // chunk offsets kept in shared memory by the row tail (V <= 2M)
// Bin-sort resolve of the row tail (sigma-hit top-k / top-k+top-p rows): the outliers are counted
// into kNB equal-width key bins while they are staged; the bins from the one holding the k-th key
// upward (<= kCapC candidates) are counting-sorted, each bin ordered in place (<= kMaxBin entries).
constexpr int kLogNB = 10;
constexpr int kNB = 1 << kLogNB;
constexpr int kCapC = 2048;
constexpr int kMaxBin = 64;
// Shared-memory work area behind the staged outliers: the bin-sort layout (counts, cursors, two
// candidate arrays) or the pivot-search layout (survivors, active sets), whichever is larger.
constexpr int kWorkBytesSearch = kCapS * 16 + kCapA * 12;
constexpr int kWorkBytesBins = kNB * 8 + kCapC * 16;
constexpr int kWorkBytes = kWorkBytesSearch > kWorkBytesBins ? kWorkBytesSearch : kWorkBytesBins;
static_assert((kMaxTailChunks + 1) * 4 <= kCapC * 8, "chunk offsets alias the candidate array");

enum Mode : int32_t { MODE_INVALID = -1, MODE_PASS = 0, MODE_TOPK = 1, MODE_TOPP = 2, MODE_TOPKP = 3 };
// ST_TP_KCAP: vocab-sharded call, a top-k row's k exceeds the k_cap the caller declared
enum Status : int32_t { ST_BAD_K = 1, ST_BAD_P = 2, ST_NONFINITE = 4, ST_TP_KCAP = 8 };

// ------------------------------------------------------------------------------------------------
// Workspace records
// ------------------------------------------------------------------------------------------------
struct alignas(16) RowPlan {
  uint32_t key_thr;   // outlier iff key >= key_thr
  int32_t mode;
  int64_t k;
  double p;
  double mu, sigma, t;
  Fx t_p;             // smallest exact mass whose fsum is >= p
  Fx t_sp;            // smallest exact mass whose fsum is >= succ(p), i.e. > p
  int32_t has_thr;    // 0: no outliers gathered for this row
  int32_t bsh;        // key-bin shift of the fused kernel's streaming histogram (provisional range)
  int32_t pad[2];
};
static_assert(sizeof(RowPlan) % 16 == 0, "RowPlan is copied with 16-byte loads");

// Per-row aggregate of the streaming pass, initialised by qrita_prep and updated with atomics by
// every chunk of the row (qrita_stream): outliers appended so far, row max / min order keys, first
// non-finite column, overflow flag, chunks finished (the row tail starts when done == nchunks).
struct alignas(16) RowAgg {
  uint32_t count;     // outliers of the row (entries beyond the row buffer are dropped)
  uint32_t maxkey;
  uint32_t minkey;
  uint32_t nf_col;    // first non-finite column, or 0xffffffff
  uint32_t ovf;       // some chunk had more outliers than its shared-memory staging holds
  uint32_t done;      // chunks finished (released after their outliers and output are written)
  uint32_t pad[2];
};

// numpy's pairwise-summation tree for the sigma sample (n = min(sample_size, V)), built on the host
// once per call: leaves (<= 128 elements each) and internal nodes grouped by height, so the device
// evaluates it level by level in parallel.  n_leaves == 0 means "too large, replay serially".
constexpr int kPwMaxLeaves = 128;
constexpr int kPwStage = 6144;  // samples staged in shared memory by qrita_prep
struct PwTree {
  int32_t n;
  int16_t n_leaves, n_internal, n_levels, pad;
  uint16_t leaf_off[kPwMaxLeaves];
  uint16_t leaf_len[kPwMaxLeaves];
  uint8_t left[kPwMaxLeaves];     // children (node ids: leaves 0.., internal nodes n_leaves..)
  uint8_t right[kPwMaxLeaves];
  uint8_t level_end[16];          // internal nodes [level_end[h-1], level_end[h]) have height h+1
};

struct Params {
  const void *logits;
  int64_t ld_in;
  void *out;
  int64_t ld_out;
  int B, V, dtype, flags, sample_size;
  const int64_t *k;
  const double *p;
  int32_t *kept_count;
  qrita_row_metrics *metrics;
  int32_t *kept_idx;        // [B][ld_idx] kept columns (unordered), or NULL; out may be NULL (index-only)
  int64_t ld_idx;
  // workspace
  RowPlan *plans;
  RowAgg *agg;              // [B]
  uint32_t *cand_bits;      // [B][xcap] outliers of each row (fp32 bits), in chunk-completion order
  uint32_t *cand_idx;       // [B][xcap] their column indices
  int32_t *status;
  int32_t *nf_col;
  int32_t *handled;         // [B] row finished by qrita_topp16 (bf16 top-p-only rows)
  int topp16;               // qrita_topp16 ran before the fused kernel: skip the rows it handled
  unsigned long long *dbg;  // [B][16] phase timestamps of the row tail (QRITA_DEBUG_TIMING)
  int nchunks;
  int total_items;
  int xcap;                 // row_cap(V)
  PwTree tree;
};

// Layout: [status[B] | nf_col[B] | dbg | plans[B] | row aggregates[B] | row outlier buffers].  Every
// record is rewritten by each call (no state carries over), and the status block only depends on
// B, so qrita_get_status needs no V.
struct WsLayout {
  size_t status, nf_col, dbg, plans, agg, handled, cand_bits, cand_idx, total;
};

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// One-time launch setup per device: the dynamic shared-memory opt-in (cudaFuncSetAttribute) and the
// occupancy-derived grid size belong to a device context, so they are cached per device ordinal.
// `slots[dev]` holds the cached value (0 = not yet set up); concurrent first calls may both run
// `init` (it is idempotent), and the value is published with release / acquire ordering.
constexpr int kMaxDevices = 64;
template <typename F>
inline cudaError_t per_device_once(int *slots, F &&init, int &out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  int v = __atomic_load_n(&slots[dev], __ATOMIC_ACQUIRE);
  if (v == 0) {
    e = init(dev, v);
    if (e != cudaSuccess) return e;
    __atomic_store_n(&slots[dev], v, __ATOMIC_RELEASE);
  }
  out = v;
  return cudaSuccess;
}

// Outlier buffer entries per row: a row never has more outliers than columns.
inline __host__ __device__ int row_cap(int V) { return V < kCapX ? V : kCapX; }

inline WsLayout ws_layout(int B, int V) {
  WsLayout L;
  const size_t cap = (size_t)row_cap(V);
  size_t off = 0;
  L.status = off;    off = align_up(off + 4ull * (size_t)B, 256);
  L.nf_col = off;    off = align_up(off + 4ull * (size_t)B, 256);
  L.dbg = off;       off = align_up(off + 128ull * (size_t)B, 256);
  L.plans = off;     off = align_up(off + sizeof(RowPlan) * (size_t)B, 256);
  L.agg = off;       off = align_up(off + sizeof(RowAgg) * (size_t)B, 256);
  L.handled = off;   off = align_up(off + 4ull * (size_t)B, 256);
  L.cand_bits = off; off = align_up(off + 4ull * (size_t)B * cap, 256);
  L.cand_idx = off;  off = align_up(off + 4ull * (size_t)B * cap, 256);
  L.total = off;
  return L;
}


cudaError_t launch_f32(const Params &P, cudaStream_t st, bool vec, cudaEvent_t prep_done,
                       cudaEvent_t stream_done);
cudaError_t launch_bf16(const Params &P, cudaStream_t st, bool vec, cudaEvent_t prep_done,
                        cudaEvent_t stream_done);

}  // namespace qrita
