// qrita_capi.cu — the extern "C" entry points of libqrita_b200.so (include/qrita_b200.h).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "qrita_types.cuh"

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

int qrita_topk_topp_ex(const void *logits, int64_t ld_in, int dtype, int B, int V,
                       const int64_t *k, const double *p, void *out, int64_t ld_out,
                       int32_t *kept_count, qrita_row_metrics *metrics,
                       void *workspace, size_t ws_bytes, int flags, int sample_size,
                       qrita_stream_t stream, void *prep_done_event, void *stream_done_event) {
  if (!logits || !out || !k || !p || !workspace) return QRITA_EINVAL_ARG;
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
  P.plans = (RowPlan *)(ws + L.plans);
  P.agg = (RowAgg *)(ws + L.agg);
  P.cand_bits = (uint32_t *)(ws + L.cand_bits);
  P.cand_idx = (uint32_t *)(ws + L.cand_idx);
  P.status = (int32_t *)(ws + L.status);
  P.nf_col = (int32_t *)(ws + L.nf_col);
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

int qrita_get_status(const void *workspace, int B, int *row, int *col, qrita_stream_t stream) {
  if (!workspace || B < 1) return QRITA_EINVAL_ARG;
  if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return QRITA_ECUDA;
  const WsLayout L = ws_layout(B, 1);  // status block offsets depend on B only
  const uint8_t *ws = (const uint8_t *)workspace;
  int32_t *st = (int32_t *)malloc(sizeof(int32_t) * 2 * (size_t)B);
  if (!st) return QRITA_EINVAL_ARG;
  if (cudaMemcpy(st, ws + L.status, sizeof(int32_t) * (size_t)B, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(st + B, ws + L.nf_col, sizeof(int32_t) * (size_t)B, cudaMemcpyDeviceToHost) != cudaSuccess) {
    free(st);
    return QRITA_ECUDA;
  }
  int code = QRITA_OK;
  if (row) *row = -1;
  if (col) *col = -1;
  for (int pass = 0; pass < 3 && code == QRITA_OK; ++pass) {
    const int bit = pass == 0 ? ST_NONFINITE : pass == 1 ? ST_BAD_K : ST_BAD_P;
    for (int r = 0; r < B; ++r) {
      if (st[r] & bit) {
        code = pass == 0 ? QRITA_ENONFINITE : pass == 1 ? QRITA_EINVAL_K : QRITA_EINVAL_P;
        if (row) *row = r;
        if (col) *col = pass == 0 ? st[B + r] : -1;
        break;
      }
    }
  }
  free(st);
  return code;
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
