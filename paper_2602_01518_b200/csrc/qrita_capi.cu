// qrita_capi.cu — the extern "C" entry points of libqrita_b200.so (include/qrita_b200.h).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <functional>
#include <thread>
#include <vector>

#include "qrita_types.cuh"
#include "qrita_internal.h"

// ================================================================================================
// C ABI (include/qrita_b200.h)
// ================================================================================================
using namespace qrita;

namespace {

struct PwNode {
  int off, len, height, left, right;
};

// Builds numpy's pairwise tree (leaf: len <= 128; split n2 = n/2 rounded down to a multiple of 8).
int pw_build(int off, int len, std::vector<PwNode> &leaves, std::vector<PwNode> &inner) {
  if (len <= 128) {
    leaves.push_back(PwNode{off, len, 0, -1, -1});
    return (int)leaves.size() - 1;          // leaf ids are provisional: leaves are numbered in order
  }
  int n2 = len / 2;
  n2 -= n2 % 8;
  const int l = pw_build(off, n2, leaves, inner);
  const bool l_leaf = n2 <= 128;
  const int r = pw_build(off + n2, len - n2, leaves, inner);
  const bool r_leaf = (len - n2) <= 128;
  const int hl = l_leaf ? 0 : inner[l].height, hr = r_leaf ? 0 : inner[r].height;
  inner.push_back(PwNode{off, len, 1 + (hl > hr ? hl : hr), l_leaf ? l : -2 - l, r_leaf ? r : -2 - r});
  return (int)inner.size() - 1;
}

void pw_tree(int n, PwTree &t) {
  memset(&t, 0, sizeof(t));
  t.n = n;
  if (n > kPwStage) return;
  std::vector<PwNode> leaves, inner;
  pw_build(0, n, leaves, inner);
  if ((int)leaves.size() > kPwMaxLeaves) return;
  const int nl = (int)leaves.size();
  // order internal nodes by height (stable) and assign ids nl + position
  std::vector<int> order(inner.size());
  for (size_t i = 0; i < inner.size(); ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return inner[a].height < inner[b].height; });
  std::vector<int> id_of(inner.size());
  for (size_t pos = 0; pos < order.size(); ++pos) id_of[order[pos]] = nl + (int)pos;
  auto child_id = [&](int c) { return c >= 0 ? c : id_of[-2 - c]; };
  for (int i = 0; i < nl; ++i) {
    t.leaf_off[i] = (uint16_t)leaves[i].off;
    t.leaf_len[i] = (uint16_t)leaves[i].len;
  }
  int levels = 0;
  for (size_t pos = 0; pos < order.size(); ++pos) {
    const PwNode &nd = inner[order[pos]];
    t.left[pos] = (uint8_t)child_id(nd.left);
    t.right[pos] = (uint8_t)child_id(nd.right);
    if (nd.height > levels) levels = nd.height;
    t.level_end[nd.height - 1] = (uint8_t)(pos + 1);
  }
  t.n_leaves = (int16_t)nl;
  t.n_internal = (int16_t)inner.size();
  t.n_levels = (int16_t)levels;
}

// Host-buffer pipeline (qrita_topk_topp_host): scratch = [chunk workspaces | k | p | in | out].
// Equal chunks of R rows (the last one shorter).  A ramp (small first / last chunks) was measured
// and lost: every copy has a fixed cost and both PCIe directions run at ~42 GB/s when busy together.
std::vector<std::pair<int, int>> host_chunks(int B, int R) {
  std::vector<std::pair<int, int>> ch;
  for (int r0 = 0; r0 < B; r0 += R) ch.push_back({r0, std::min(R, B - r0)});
  return ch;
}

struct HostLayout {
  int nchunks;
  std::vector<std::pair<int, int>> chunks;  // (first row, rows)
  size_t ws_each, st, nf, k, p, in, out, total;
};

HostLayout host_layout(int B, int V, int dtype, int chunk_rows) {
  HostLayout H;
  const size_t es = dtype == QRITA_DTYPE_F32 ? 4 : 2;
  H.chunks = host_chunks(B, chunk_rows);
  H.nchunks = (int)H.chunks.size();
  H.ws_each = align_up(ws_layout(chunk_rows, V).total, 256);
  size_t off = H.ws_each * (size_t)H.nchunks;
  H.st = off;  off = align_up(off + 4ull * (size_t)B, 256);
  H.nf = off;  off = align_up(off + 4ull * (size_t)B, 256);
  H.k = off;   off = align_up(off + 8ull * (size_t)B, 256);
  H.p = off;   off = align_up(off + 8ull * (size_t)B, 256);
  H.in = off;  off = align_up(off + es * (size_t)B * (size_t)V, 256);
  H.out = off; off = align_up(off + es * (size_t)B * (size_t)V, 256);
  H.total = off;
  return H;
}

// The library's own streams and a growing event pool, per device; one host-buffer call enqueues at a
// time (the events are reused across calls, so the enqueue section is serialised).  Pageable host
// buffers are staged through two page-locked slots per direction (grown on demand).
struct HostPipe {
  cudaStream_t up = nullptr, comp = nullptr, down = nullptr;
  std::vector<cudaEvent_t> ev;
  void *stage_in[2] = {nullptr, nullptr}, *stage_out[2] = {nullptr, nullptr};
  size_t stage_bytes = 0;
  cudaEvent_t in_free[2] = {nullptr, nullptr}, out_ready[2] = {nullptr, nullptr};
  int32_t *kept_host = nullptr;  // sparse downloads: kept columns [B][kcap] | counts [B] (page-locked)
  size_t kept_host_bytes = 0;
};
std::mutex g_host_mu;
HostPipe g_host_pipe[64];

cudaError_t host_pipe_get(int dev, size_t nev, HostPipe *&hp) {
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  hp = &g_host_pipe[dev];
  cudaError_t e = cudaSuccess;
  for (cudaStream_t *s : {&hp->up, &hp->comp, &hp->down})
    if (!*s && (e = cudaStreamCreateWithFlags(s, cudaStreamNonBlocking)) != cudaSuccess) return e;
  while (hp->ev.size() < nev) {
    cudaEvent_t x;
    if ((e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming)) != cudaSuccess) return e;
    hp->ev.push_back(x);
  }
  for (int i = 0; i < 2; ++i)
    for (cudaEvent_t *x : {&hp->in_free[i], &hp->out_ready[i]})
      if (!*x && (e = cudaEventCreateWithFlags(x, cudaEventDisableTiming)) != cudaSuccess) return e;
  return cudaSuccess;
}

cudaError_t host_stage_reserve(HostPipe *hp, size_t bytes) {
  if (hp->stage_bytes >= bytes) return cudaSuccess;
  for (int i = 0; i < 2; ++i) {
    // the slots may still feed copies of the previous call
    if (hp->in_free[i]) cudaEventSynchronize(hp->in_free[i]);
    if (hp->out_ready[i]) cudaEventSynchronize(hp->out_ready[i]);
    for (void **b : {&hp->stage_in[i], &hp->stage_out[i]}) {
      if (*b) cudaFreeHost(*b);
      *b = nullptr;
    }
  }
  hp->stage_bytes = 0;
  for (int i = 0; i < 2; ++i)
    for (void **b : {&hp->stage_in[i], &hp->stage_out[i]}) {
      cudaError_t e = cudaHostAlloc(b, bytes, cudaHostAllocPortable);
      if (e != cudaSuccess) return e;
    }
  hp->stage_bytes = bytes;
  return cudaSuccess;
}

// Parallel host memcpy for the pageable staging copies: a persistent pool of worker threads (the
// calling thread helps); one copy at a time.  QRITA_HOST_COPY_THREADS overrides the thread count.
class CopyPool {
 public:
  static CopyPool &get() {
    static CopyPool *pool = new CopyPool();  // never destroyed: its threads end with the process
    return *pool;
  }
  // fn(0 .. n-1) over every thread of the pool (items claimed one at a time; the caller helps)
  void parallel_for(size_t n, const std::function<void(size_t)> &fn) {
    if (n < 2 || nthreads_ == 0) {
      for (size_t i = 0; i < n; ++i) fn(i);
      return;
    }
    std::lock_guard<std::mutex> call(call_mu_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      items_ = n;
      next_.store(0);
      limit_ = nthreads_;
      active_ = nthreads_;
      ++gen_;
    }
    cv_work_.notify_all();
    run_pieces();
    std::unique_lock<std::mutex> lk(mu_);
    cv_done_.wait(lk, [&] { return active_ == 0; });
    fn_ = nullptr;
  }
  // memcpy over `copiers_` threads (more compete with the DMA for host memory bandwidth)
  void copy(void *d, const void *s, size_t n) {
    if (n < (1u << 20) || copiers_ == 0) {
      memcpy(d, s, n);
      return;
    }
    std::lock_guard<std::mutex> call(call_mu_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = nullptr;
      dst_ = (uint8_t *)d;
      src_ = (const uint8_t *)s;
      bytes_ = n;
      size_t piece = n / (size_t)(4 * (copiers_ + 1));
      piece = std::max<size_t>(piece, 256u << 10);
      piece_ = (piece + 4095) & ~(size_t)4095;
      next_.store(0);
      limit_ = copiers_;
      active_ = copiers_;
      ++gen_;
    }
    cv_work_.notify_all();
    run_pieces();
    std::unique_lock<std::mutex> lk(mu_);
    cv_done_.wait(lk, [&] { return active_ == 0; });
  }

 private:
  CopyPool() {
    // copies: half the hardware threads, at most 8 — measured best on the 16-core B200 host (cfg2
    // run_batch 5.0 ms with 8 copiers vs 6.5 ms with 16, tools/e2e_pageable.py); host-built rows of
    // sparse downloads: every hardware thread (2.98 ms with 8, 2.77-2.83 with 12-16,
    // tools/e2e_sparse_sweep.py)
    const int hw = std::max(1, (int)std::thread::hardware_concurrency());
    int c = std::min(8, std::max(1, hw / 2)), t = hw;
    if (const char *ev = getenv("QRITA_HOST_COPY_THREADS")) c = atoi(ev);
    if (const char *ev = getenv("QRITA_HOST_BUILD_THREADS")) t = atoi(ev);
    copiers_ = std::max(0, std::min(c, 32) - 1);  // the caller is one of them
    nthreads_ = std::max(copiers_, std::max(0, std::min(t, 32) - 1));
    for (int i = 0; i < nthreads_; ++i) std::thread([this, i] { worker(i); }).detach();
  }
  void run_pieces() {
    if (fn_) {
      for (size_t i; (i = next_.fetch_add(1)) < items_;) (*fn_)(i);
      return;
    }
    for (;;) {
      const size_t off = next_.fetch_add(1) * piece_;
      if (off >= bytes_) return;
      memcpy(dst_ + off, src_ + off, std::min(piece_, bytes_ - off));
    }
  }
  void worker(int id) {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      cv_work_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      if (id >= limit_) continue;  // not part of this job
      lk.unlock();
      run_pieces();
      lk.lock();
      if (--active_ == 0) cv_done_.notify_all();
    }
  }
  std::mutex call_mu_, mu_;
  std::condition_variable cv_work_, cv_done_;
  int nthreads_ = 0, copiers_ = 0, limit_ = 0, active_ = 0;
  uint64_t gen_ = 0;
  uint8_t *dst_ = nullptr;
  const uint8_t *src_ = nullptr;
  size_t bytes_ = 0, piece_ = 0, items_ = 0;
  const std::function<void(size_t)> *fn_ = nullptr;
  std::atomic<size_t> next_{0};
};

// Sparse downloads (host pipeline): when every row keeps at most k < V entries (top-k active, k small),
// the kernel writes each row's kept columns instead of the masked row; only those come back over
// PCIe and the host builds the masked rows from its own copy of the logits (-inf fill + copy of the
// kept entries, bit-identical).  Returns the kept-column slots per row (a multiple of 4), or 0 when
// the batch is not eligible.
constexpr int64_t kSparseCap = 4096;
int sparse_slots(int B, int V, int dtype, const int64_t *k_host) {
  int64_t kmax = 0;
  for (int r = 0; r < B; ++r) {
    const int64_t k = k_host[r];
    if (!(k >= 1 && k < (int64_t)V)) return 0;  // top-p-only / pass-through / invalid rows: dense
    kmax = k > kmax ? k : kmax;
  }
  const int64_t slots = (kmax + 3) & ~(int64_t)3;
  const int64_t es = dtype == QRITA_DTYPE_F32 ? 4 : 2;
  if (slots > kSparseCap || (slots + 1) * 4 > (int64_t)V * es) return 0;  // kept columns fit the out rows
  return (int)slots;
}

bool is_pinned(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Sparse or dense downloads for a host-buffer call (measured, tools/e2e_sparse_sweep.py /
// tools/e2e_pageable.py): sparse whenever eligible, except for a pageable input with a page-locked
// output, where the host threads are busy staging the input and the DMA delivers the dense rows
// faster than they could build them.
int host_slots(int B, int V, int dtype, const int64_t *k_host, const void *in_host, const void *out_host) {
  if (getenv("QRITA_HOST_DENSE")) return 0;
  const bool force = getenv("QRITA_HOST_SPARSE") != nullptr;
  if (!force && in_host && out_host && !is_pinned(in_host) && is_pinned(out_host)) return 0;
  return sparse_slots(B, V, dtype, k_host);
}

}  // namespace

extern "C" {

size_t qrita_workspace_bytes(int B, int V, int dtype, int flags) {
  (void)dtype; (void)flags;
  if (B < 1 || V < 1) return 0;
  return ws_layout(B, V).total;
}

int qrita_workspace_init(void *workspace, size_t ws_bytes, qrita_stream_t stream) {
  if (!workspace) return QRITA_EINVAL_ARG;
  return cudaMemsetAsync(workspace, 0, ws_bytes, (cudaStream_t)stream) == cudaSuccess ? QRITA_OK : QRITA_ECUDA;
}

int qrita_topk_topp(const void *logits, int64_t ld_in, int dtype, int B, int V,
                    const int64_t *k, const double *p, void *out, int64_t ld_out,
                    int32_t *kept_count, qrita_row_metrics *metrics,
                    void *workspace, size_t ws_bytes, int flags, int sample_size,
                    qrita_stream_t stream) {
  return qrita_topk_topp_ex(logits, ld_in, dtype, B, V, k, p, out, ld_out, kept_count, metrics,
                            workspace, ws_bytes, flags, sample_size, stream, NULL, NULL);
}

}  // extern "C"

namespace qrita {

// numpy's pairwise-sum tree over the first n elements (the sigma plan's sample), for other TUs
void pw_tree_build(int n, PwTree &t) { pw_tree(n, t); }

// qrita_topk_topp_ex with the status / nf_col words optionally placed outside the workspace (the
// host-buffer pipeline gathers the chunks' status into one [B] block).
int topk_topp_impl(const void *logits, int64_t ld_in, int dtype, int B, int V, const int64_t *k, const double *p,
                   void *out, int64_t ld_out, int32_t *kept_count, qrita_row_metrics *metrics, void *workspace,
                   size_t ws_bytes, int flags, int sample_size, qrita_stream_t stream, void *prep_done_event,
                   void *stream_done_event, int32_t *status, int32_t *nf_col, int32_t *kept_idx,
                   int64_t ld_idx) {
  if (!logits || !k || !p || !workspace) return QRITA_EINVAL_ARG;
  if (!out && !kept_idx) return QRITA_EINVAL_ARG;
  if (kept_idx && (ld_idx < 1 || (!kept_count && !metrics))) return QRITA_EINVAL_ARG;
  if (!out) {
    if (flags & QRITA_INPLACE) return QRITA_EINVAL_ARG;
    ld_out = V;
  }
  if (B < 1 || V < 1 || ld_in < V || ld_out < V || sample_size < 1) return QRITA_EINVAL_ARG;
  if (dtype != QRITA_DTYPE_F32 && dtype != QRITA_DTYPE_BF16) return QRITA_EINVAL_ARG;
  if (flags & ~(QRITA_SEARCH_BINARY | QRITA_NO_SIGMA | QRITA_FORCE_FALLBACK | QRITA_NO_DUP | QRITA_INPLACE |
                QRITA_DEBUG_TIMING | QRITA_STAGED))
    return QRITA_EINVAL_ARG;
  const bool inplace = (flags & QRITA_INPLACE) != 0;
  if (inplace != (logits == out)) return QRITA_EINVAL_ARG;
  if (inplace && ld_in != ld_out) return QRITA_EINVAL_ARG;
  const WsLayout L = ws_layout(B, V);
  if (ws_bytes < L.total || ((uintptr_t)workspace & 255u)) return QRITA_EWORKSPACE;
  const size_t nchunks = (size_t)((V + kChunk - 1) / kChunk);
  if ((size_t)B * nchunks > 0x7fffffffull) return QRITA_EINVAL_ARG;

  uint8_t *ws = (uint8_t *)workspace;
  Params P;
  memset(&P, 0, sizeof(P));
  P.logits = logits; P.ld_in = ld_in; P.out = out; P.ld_out = ld_out;
  P.B = B; P.V = V; P.dtype = dtype; P.flags = flags; P.sample_size = sample_size;
  P.k = k; P.p = p; P.kept_count = kept_count; P.metrics = metrics;
  P.kept_idx = kept_idx; P.ld_idx = ld_idx;
  P.plans = (RowPlan *)(ws + L.plans);
  P.agg = (RowAgg *)(ws + L.agg);
  P.handled = (int32_t *)(ws + L.handled);
  P.cand_bits = (uint32_t *)(ws + L.cand_bits);
  P.cand_idx = (uint32_t *)(ws + L.cand_idx);
  P.status = status ? status : (int32_t *)(ws + L.status);
  P.nf_col = nf_col ? nf_col : (int32_t *)(ws + L.nf_col);
  P.dbg = (unsigned long long *)(ws + L.dbg);
  P.nchunks = (int)nchunks;
  P.xcap = row_cap(V);
  P.total_items = (int)((size_t)B * nchunks);
  pw_tree(sample_size < V ? sample_size : V, P.tree);

  const size_t es = dtype == QRITA_DTYPE_F32 ? 4 : 2;
  const bool vec = ((uintptr_t)logits % 16 == 0) && ((uintptr_t)out % 16 == 0) &&
                   ((size_t)ld_in * es % 16 == 0) && ((size_t)ld_out * es % 16 == 0);
  cudaError_t e = dtype == QRITA_DTYPE_F32
                      ? launch_f32(P, (cudaStream_t)stream, vec, (cudaEvent_t)prep_done_event,
                                   (cudaEvent_t)stream_done_event)
                      : launch_bf16(P, (cudaStream_t)stream, vec, (cudaEvent_t)prep_done_event,
                                    (cudaEvent_t)stream_done_event);
  return e == cudaSuccess ? QRITA_OK : QRITA_ECUDA;
}

// First failing row of a [status[B] | nf_col[B]] pair in host memory (precedence: non-finite, k, p).
int scan_status(const int32_t *st, const int32_t *nf, int B, int *row, int *col) {
  if (row) *row = -1;
  if (col) *col = -1;
  for (int pass = 0; pass < 4; ++pass) {
    const int bit = pass == 0 ? ST_NONFINITE : pass == 1 ? ST_BAD_K : pass == 2 ? ST_BAD_P : ST_TP_KCAP;
    for (int r = 0; r < B; ++r) {
      if (st[r] & bit) {
        if (row) *row = r;
        if (col) *col = pass == 0 ? nf[r] : -1;
        return pass == 0 ? QRITA_ENONFINITE : pass == 1 ? QRITA_EINVAL_K : pass == 2 ? QRITA_EINVAL_P
                                                                                  : QRITA_EINVAL_ARG;
      }
    }
  }
  return QRITA_OK;
}

int read_status(const int32_t *st_dev, const int32_t *nf_dev, int B, int *row, int *col, qrita_stream_t stream) {
  if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return QRITA_ECUDA;
  std::vector<int32_t> st(2 * (size_t)B);
  if (cudaMemcpy(st.data(), st_dev, sizeof(int32_t) * (size_t)B, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(st.data() + B, nf_dev, sizeof(int32_t) * (size_t)B, cudaMemcpyDeviceToHost) != cudaSuccess)
    return QRITA_ECUDA;
  return scan_status(st.data(), st.data() + B, B, row, col);
}

}  // namespace qrita

extern "C" {

int qrita_topk_topp_ex(const void *logits, int64_t ld_in, int dtype, int B, int V,
                       const int64_t *k, const double *p, void *out, int64_t ld_out,
                       int32_t *kept_count, qrita_row_metrics *metrics,
                       void *workspace, size_t ws_bytes, int flags, int sample_size,
                       qrita_stream_t stream, void *prep_done_event, void *stream_done_event) {
  return topk_topp_impl(logits, ld_in, dtype, B, V, k, p, out, ld_out, kept_count, metrics, workspace, ws_bytes,
                        flags, sample_size, stream, prep_done_event, stream_done_event, NULL, NULL);
}

int qrita_topk_topp_idx(const void *logits, int64_t ld_in, int dtype, int B, int V, const int64_t *k,
                        const double *p, void *out, int64_t ld_out, int32_t *kept_idx, int64_t ld_idx,
                        int32_t *kept_count, qrita_row_metrics *metrics, void *workspace, size_t ws_bytes,
                        int flags, int sample_size, qrita_stream_t stream) {
  if (kept_idx && ld_idx < V) return QRITA_EINVAL_ARG;  // a row may keep all V columns
  return topk_topp_impl(logits, ld_in, dtype, B, V, k, p, out, ld_out, kept_count, metrics, workspace, ws_bytes,
                        flags, sample_size, stream, NULL, NULL, NULL, NULL, kept_idx, ld_idx);
}

size_t qrita_host_scratch_bytes(int B, int V, int dtype, int chunk_rows) {
  if (B < 1 || V < 1 || chunk_rows < 1) return 0;
  return host_layout(B, V, dtype, chunk_rows < B ? chunk_rows : B).total;
}

int qrita_topk_topp_host(const void *logits_host, int dtype, int B, int V,
                         const int64_t *k_host, const double *p_host, void *out_host,
                         int32_t *kept_count, qrita_row_metrics *metrics,
                         void *scratch, size_t scratch_bytes, int chunk_rows, int flags, int sample_size,
                         qrita_stream_t stream) {
  if (!logits_host || !out_host || !k_host || !p_host || !scratch) return QRITA_EINVAL_ARG;
  if (B < 1 || V < 1 || chunk_rows < 1 || sample_size < 1) return QRITA_EINVAL_ARG;
  if (dtype != QRITA_DTYPE_F32 && dtype != QRITA_DTYPE_BF16) return QRITA_EINVAL_ARG;
  if (flags & (QRITA_INPLACE | QRITA_DEBUG_TIMING)) return QRITA_EINVAL_ARG;
  if (chunk_rows > B) chunk_rows = B;
  const HostLayout H = host_layout(B, V, dtype, chunk_rows);
  if (scratch_bytes < H.total || ((uintptr_t)scratch & 255u)) return QRITA_EWORKSPACE;
  const size_t es = dtype == QRITA_DTYPE_F32 ? 4 : 2;
  const size_t row_bytes = es * (size_t)V;
  uint8_t *sc = (uint8_t *)scratch;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return QRITA_ECUDA;
  std::lock_guard<std::mutex> lock(g_host_mu);
  HostPipe *hp = nullptr;
  const size_t nc = (size_t)H.nchunks;
  if (host_pipe_get(dev, 3 * nc + 4, hp) != cudaSuccess) return QRITA_ECUDA;
  cudaEvent_t *landed = hp->ev.data(), *done = landed + nc, *ev0 = done + nc, *fetched = ev0 + 4;
  const int slots = host_slots(B, V, dtype, k_host, logits_host, out_host);  // > 0: sparse downloads
  int32_t *kidx_d = (int32_t *)(sc + H.out), *cnt_d = kidx_d + (size_t)B * slots;
  const cudaStream_t caller = (cudaStream_t)stream;
  auto ok = [](cudaError_t e) { return e == cudaSuccess; };
  // QRITA_HOST_TRACE: timing events per chunk (uploaded / truncated / downloaded), printed to stderr
  const bool trace = getenv("QRITA_HOST_TRACE") != NULL;
  std::vector<cudaEvent_t> tr(trace ? 3 * nc + 1 : 0);
  for (auto &x : tr) cudaEventCreate(&x);
  if (trace) cudaEventRecord(tr[3 * nc], caller);
  // everything already on the caller's stream (buffers, kept_count / metrics) comes first
  // ... and so does the previous host-buffer call on these streams (its buffers may be this call's):
  // ev0[1] still holds its last download (a never-recorded event is complete)
  if (!ok(cudaEventRecord(ev0[0], caller))) return QRITA_ECUDA;
  for (cudaStream_t s : {hp->up, hp->comp, hp->down})
    if (!ok(cudaStreamWaitEvent(s, ev0[0], 0)) || !ok(cudaStreamWaitEvent(s, ev0[1], 0))) return QRITA_ECUDA;
  // chunk workspaces start clean (one memset, overlapping the first upload)
  if (!ok(cudaMemsetAsync(sc, 0, H.ws_each * nc, hp->comp))) return QRITA_ECUDA;
  if (!ok(cudaMemcpyAsync(sc + H.k, k_host, 8ull * (size_t)B, cudaMemcpyHostToDevice, hp->up)) ||
      !ok(cudaMemcpyAsync(sc + H.p, p_host, 8ull * (size_t)B, cudaMemcpyHostToDevice, hp->up)))
    return QRITA_ECUDA;
  // Page-locked host buffers: every upload is enqueued up front, then the kernels and downloads.
  // Pageable buffers: the host copies each chunk into a page-locked slot (CopyPool, many threads)
  // right before its upload, and each downloaded chunk out of its slot one chunk later, so the DMA
  // of chunk c overlaps the host copies of chunks c +- 1.
  const bool in_staged = !is_pinned(logits_host), out_staged = !slots && !is_pinned(out_host);
  if (slots) {
    const size_t need = (size_t)B * (slots + 1) * 4;
    if (hp->kept_host_bytes < need) {
      if (hp->kept_host) cudaFreeHost(hp->kept_host);
      hp->kept_host = nullptr;
      hp->kept_host_bytes = 0;
      if (!ok(cudaHostAlloc((void **)&hp->kept_host, need, cudaHostAllocPortable))) return QRITA_ECUDA;
      hp->kept_host_bytes = need;
    }
  }
  // sparse: the masked rows of chunk c, built on the host from the input and the kept columns
  // -inf background of chunk c's rows: needs nothing from the GPU, so it runs while the chunk is
  // still uploading / being truncated
  auto fill = [&](size_t c) {
    const size_t r0 = (size_t)H.chunks[c].first, nr = (size_t)H.chunks[c].second;
    CopyPool::get().parallel_for(nr, [&](size_t i) {
      uint8_t *o = (uint8_t *)out_host + (r0 + i) * row_bytes;
      if (es == 4) std::fill_n((uint32_t *)o, (size_t)V, 0xff800000u);
      else std::fill_n((uint16_t *)o, (size_t)V, (uint16_t)0xff80u);
    });
  };
  // the kept entries of chunk c, copied from the host's own logits once its kept columns are back
  auto scatter = [&](size_t c) -> bool {
    const size_t r0 = (size_t)H.chunks[c].first, nr = (size_t)H.chunks[c].second;
    if (!ok(cudaEventSynchronize(fetched[c]))) return false;
    const int32_t *kh = hp->kept_host, *ch = hp->kept_host + (size_t)B * slots;
    CopyPool::get().parallel_for(nr, [&](size_t i) {
      const size_t r = r0 + i;
      const int32_t n = std::max(0, std::min(ch[r], slots));  // invalid rows: whatever came back
      const int32_t *cols = kh + r * (size_t)slots;
      if (es == 4) {
        uint32_t *o = (uint32_t *)((uint8_t *)out_host + r * row_bytes);
        const uint32_t *x = (const uint32_t *)((const uint8_t *)logits_host + r * row_bytes);
        for (int32_t j = 0; j < n; ++j)
          if ((uint32_t)cols[j] < (uint32_t)V) o[cols[j]] = x[cols[j]];
      } else {
        uint16_t *o = (uint16_t *)((uint8_t *)out_host + r * row_bytes);
        const uint16_t *x = (const uint16_t *)((const uint8_t *)logits_host + r * row_bytes);
        for (int32_t j = 0; j < n; ++j)
          if ((uint32_t)cols[j] < (uint32_t)V) o[cols[j]] = x[cols[j]];
      }
    });
    return true;
  };
  if ((in_staged || out_staged) &&
      host_stage_reserve(hp, (size_t)H.chunks[0].second * row_bytes) != cudaSuccess)
    return QRITA_ECUDA;
  auto upload = [&](size_t c) -> bool {
    const size_t r0 = (size_t)H.chunks[c].first, nr = (size_t)H.chunks[c].second;
    const uint8_t *src = (const uint8_t *)logits_host + r0 * row_bytes;
    if (in_staged) {
      const int slot = (int)(c & 1);
      if (!ok(cudaEventSynchronize(hp->in_free[slot]))) return false;  // its previous upload is done
      CopyPool::get().copy(hp->stage_in[slot], src, nr * row_bytes);
      src = (const uint8_t *)hp->stage_in[slot];
    }
    if (!ok(cudaMemcpyAsync(sc + H.in + r0 * row_bytes, src, nr * row_bytes, cudaMemcpyHostToDevice, hp->up)) ||
        !ok(cudaEventRecord(landed[c], hp->up)))
      return false;
    if (in_staged && !ok(cudaEventRecord(hp->in_free[c & 1], hp->up))) return false;
    if (trace) cudaEventRecord(tr[c], hp->up);
    return true;
  };
  auto drain = [&](size_t c) -> bool {  // staged output: chunk c from its slot to the caller's buffer
    const size_t r0 = (size_t)H.chunks[c].first, nr = (size_t)H.chunks[c].second;
    if (!ok(cudaEventSynchronize(hp->out_ready[c & 1]))) return false;
    CopyPool::get().copy((uint8_t *)out_host + r0 * row_bytes, hp->stage_out[c & 1], nr * row_bytes);
    return true;
  };
  if (!in_staged)
    for (size_t c = 0; c < nc; ++c)
      if (!upload(c)) return QRITA_ECUDA;
  for (size_t c = 0; c < nc; ++c) {
    const size_t r0 = (size_t)H.chunks[c].first, nr = (size_t)H.chunks[c].second;
    if (in_staged && !upload(c)) return QRITA_ECUDA;
    if (!ok(cudaStreamWaitEvent(hp->comp, landed[c], 0))) return QRITA_ECUDA;
    const int rc = slots
        ? topk_topp_impl(sc + H.in + r0 * row_bytes, V, dtype, (int)nr, V, (const int64_t *)(sc + H.k) + r0,
                         (const double *)(sc + H.p) + r0, NULL, V, cnt_d + r0, metrics ? metrics + r0 : NULL,
                         sc + c * H.ws_each, H.ws_each, flags, sample_size, (qrita_stream_t)hp->comp, NULL, NULL,
                         (int32_t *)(sc + H.st) + r0, (int32_t *)(sc + H.nf) + r0, kidx_d + r0 * (size_t)slots,
                         slots)
        : topk_topp_impl(sc + H.in + r0 * row_bytes, V, dtype, (int)nr, V, (const int64_t *)(sc + H.k) + r0,
                         (const double *)(sc + H.p) + r0, sc + H.out + r0 * row_bytes, V,
                         kept_count ? kept_count + r0 : NULL, metrics ? metrics + r0 : NULL, sc + c * H.ws_each,
                         H.ws_each, flags, sample_size, (qrita_stream_t)hp->comp, NULL, NULL,
                         (int32_t *)(sc + H.st) + r0, (int32_t *)(sc + H.nf) + r0);
    if (rc != QRITA_OK) return rc;
    if (trace) cudaEventRecord(tr[nc + c], hp->comp);
    if (!ok(cudaEventRecord(done[c], hp->comp)) || !ok(cudaStreamWaitEvent(hp->down, done[c], 0)))
      return QRITA_ECUDA;
    if (slots) {
      // the chunk's kept columns and counts; the host builds chunk c - 1 meanwhile
      if (!ok(cudaMemcpyAsync(hp->kept_host + r0 * (size_t)slots, kidx_d + r0 * (size_t)slots,
                              nr * (size_t)slots * 4, cudaMemcpyDeviceToHost, hp->down)) ||
          !ok(cudaMemcpyAsync(hp->kept_host + (size_t)B * slots + r0, cnt_d + r0, nr * 4, cudaMemcpyDeviceToHost,
                              hp->down)) ||
          !ok(cudaEventRecord(fetched[c], hp->down)))
        return QRITA_ECUDA;
      if (kept_count && !ok(cudaMemcpyAsync(kept_count + r0, cnt_d + r0, nr * 4, cudaMemcpyDeviceToDevice,
                                            hp->down)))
        return QRITA_ECUDA;
      if (trace) cudaEventRecord(tr[2 * nc + c], hp->down);
      fill(c);
      if (c > 0 && !scatter(c - 1)) return QRITA_ECUDA;
      continue;
    }
    if (out_staged) {
      if (!ok(cudaMemcpyAsync(hp->stage_out[c & 1], sc + H.out + r0 * row_bytes, nr * row_bytes,
                              cudaMemcpyDeviceToHost, hp->down)) ||
          !ok(cudaEventRecord(hp->out_ready[c & 1], hp->down)))
        return QRITA_ECUDA;
      if (c > 0 && !drain(c - 1)) return QRITA_ECUDA;
    } else if (!ok(cudaMemcpyAsync((uint8_t *)out_host + r0 * row_bytes, sc + H.out + r0 * row_bytes,
                                   nr * row_bytes, cudaMemcpyDeviceToHost, hp->down))) {
      return QRITA_ECUDA;
    }
    if (trace) cudaEventRecord(tr[2 * nc + c], hp->down);
  }
  if (out_staged && !drain(nc - 1)) return QRITA_ECUDA;
  if (slots && !scatter(nc - 1)) return QRITA_ECUDA;
  if (trace) {
    cudaDeviceSynchronize();
    for (size_t c = 0; c < nc; ++c) {
      float a = 0, b = 0, d = 0;
      cudaEventElapsedTime(&a, tr[3 * nc], tr[c]);
      cudaEventElapsedTime(&b, tr[3 * nc], tr[nc + c]);
      cudaEventElapsedTime(&d, tr[3 * nc], tr[2 * nc + c]);
      fprintf(stderr, "chunk %zu: up %.3f  kernel %.3f  down %.3f ms\n", c, a, b, d);
    }
    for (auto &x : tr) cudaEventDestroy(x);
  }
  // the caller's stream waits for the downloads and the last kernel (kept_count / metrics)
  if (!ok(cudaEventRecord(ev0[1], hp->down)) || !ok(cudaEventRecord(ev0[2], hp->comp)) ||
      !ok(cudaEventRecord(ev0[3], hp->up)) || !ok(cudaStreamWaitEvent(caller, ev0[1], 0)) ||
      !ok(cudaStreamWaitEvent(caller, ev0[2], 0)) || !ok(cudaStreamWaitEvent(caller, ev0[3], 0)))
    return QRITA_ECUDA;
  return QRITA_OK;
}

int64_t qrita_host_download_bytes(int B, int V, int dtype, const int64_t *k_host, const void *logits_host,
                                  const void *out_host) {
  if (B < 1 || V < 1 || !k_host) return -1;
  const int slots = host_slots(B, V, dtype, k_host, logits_host, out_host);
  const int64_t es = dtype == QRITA_DTYPE_F32 ? 4 : 2;
  return slots ? (int64_t)B * (slots + 1) * 4 : (int64_t)B * V * es;
}

int qrita_get_status_host(const void *scratch, int B, int V, int dtype, int chunk_rows, int *row, int *col,
                          qrita_stream_t stream) {
  if (!scratch || B < 1 || V < 1 || chunk_rows < 1) return QRITA_EINVAL_ARG;
  const HostLayout H = host_layout(B, V, dtype, chunk_rows < B ? chunk_rows : B);
  const uint8_t *sc = (const uint8_t *)scratch;
  return read_status((const int32_t *)(sc + H.st), (const int32_t *)(sc + H.nf), B, row, col, stream);
}

int qrita_get_status(const void *workspace, int B, int *row, int *col, qrita_stream_t stream) {
  if (!workspace || B < 1) return QRITA_EINVAL_ARG;
  const WsLayout L = ws_layout(B, 1);  // status block offsets depend on B only
  const uint8_t *ws = (const uint8_t *)workspace;
  return read_status((const int32_t *)(ws + L.status), (const int32_t *)(ws + L.nf_col), B, row, col, stream);
}

int qrita_get_timing(const void *workspace, int B, unsigned long long *out, qrita_stream_t stream) {
  if (!workspace || !out || B < 1) return QRITA_EINVAL_ARG;
  if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return QRITA_ECUDA;
  const WsLayout L = ws_layout(B, 1);
  return cudaMemcpy(out, (const uint8_t *)workspace + L.dbg, 128ull * (size_t)B, cudaMemcpyDeviceToHost) ==
                 cudaSuccess ? QRITA_OK : QRITA_ECUDA;
}

const char *qrita_strerror(int code) {
  switch (code) {
    case QRITA_OK: return "ok";
    case QRITA_EINVAL_ARG: return "invalid argument";
    case QRITA_EINVAL_K: return "k out of range [1,V]";
    case QRITA_EINVAL_P: return "p out of range (0,1]";
    case QRITA_ENONFINITE: return "non-finite logit";
    case QRITA_EWORKSPACE: return "workspace too small or misaligned";
    case QRITA_ECUDA: return "CUDA runtime error";
    case QRITA_ENCCL: return "NCCL error";
    default: return "unknown error";
  }
}

int qrita_version(void) { return 100; }

}  // extern "C"
