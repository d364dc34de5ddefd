// qrita_capi.cu — the extern "C" entry points of libqrita_b200.so (include/qrita_b200.h).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "qrita_types.cuh"

// ================================================================================================
// C ABI (include/qrita_b200.h)
// ================================================================================================
using namespace qrita;

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
  if (!logits || !out || !k || !p || !workspace) return QRITA_EINVAL_ARG;
  if (B < 1 || V < 1 || ld_in < V || ld_out < V || sample_size < 1) return QRITA_EINVAL_ARG;
  if (dtype != QRITA_DTYPE_F32 && dtype != QRITA_DTYPE_BF16) return QRITA_EINVAL_ARG;
  if (flags & ~(QRITA_SEARCH_BINARY | QRITA_NO_SIGMA | QRITA_FORCE_FALLBACK | QRITA_NO_DUP | QRITA_INPLACE))
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
  P.cstats = (ChunkStat *)(ws + L.cstats);
  P.cand_bits = (uint32_t *)(ws + L.cand_bits);
  P.cand_idx = (uint32_t *)(ws + L.cand_idx);
  P.row_done = (uint32_t *)(ws + L.row_done);
  P.work_ctr = (uint32_t *)(ws + L.ctrs);
  P.exit_ctr = (uint32_t *)(ws + L.ctrs + 4);
  P.status = (int32_t *)(ws + L.status);
  P.nf_col = (int32_t *)(ws + L.nf_col);
  P.nchunks = (int)nchunks;
  P.total_items = (int)((size_t)B * nchunks);

  const size_t es = dtype == QRITA_DTYPE_F32 ? 4 : 2;
  const bool vec = ((uintptr_t)logits % 16 == 0) && ((uintptr_t)out % 16 == 0) &&
                   ((size_t)ld_in * es % 16 == 0) && ((size_t)ld_out * es % 16 == 0);
  cudaError_t e = dtype == QRITA_DTYPE_F32 ? launch_f32(P, (cudaStream_t)stream, vec)
                                           : launch_bf16(P, (cudaStream_t)stream, vec);
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
