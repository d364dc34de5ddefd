// qrita_prims.cu — the reference's sigma_trunc primitives as C-ABI entry points (include/qrita_b200.h):
// the embedded quantile tables (host) and row_stats (device, numpy's pairwise mean bit for bit).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "qrita_plan.cuh"

namespace qrita {

static const double h_topk_table[kTableSize] = {QRITA_TOPK_TABLE_VALUES};
static const double h_topp_table[kTableSize] = {QRITA_TOPP_TABLE_VALUES};

// sigma_trunc.py:69-82: mu = mean(x[:n]), var = mean(x*x) - mu*mu floored at 0, sigma = sqrt(var);
// numpy's pairwise sums (pairwise_serial), true division by n, no FMA.  One thread per row.
template <typename T>
__global__ void row_stats_kernel(const T *x, int64_t ld, int B, int n, double *out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= B) return;
  const T *a = x + (size_t)r * ld;
  const double s = pairwise_serial<T, false>(a, n);
  const double sq = pairwise_serial<T, true>(a, n);
  const double mu = __ddiv_rn(s, (double)n);
  const double var = __dsub_rn(__ddiv_rn(sq, (double)n), __dmul_rn(mu, mu));
  out[2 * (size_t)r] = mu;
  out[2 * (size_t)r + 1] = __dsqrt_rn(var > 0.0 ? var : 0.0);
}

}  // namespace qrita

using namespace qrita;

extern "C" {

int qrita_sigma_table(int kind, double *out, int n) {
  if (!out || n < kTableSize || (kind != 0 && kind != 1)) return QRITA_EINVAL_ARG;
  memcpy(out, kind == 0 ? h_topk_table : h_topp_table, sizeof(double) * kTableSize);
  return QRITA_OK;
}

int qrita_row_stats(const void *logits, int64_t ld, int dtype, int B, int V, int sample_size, double *out,
                    qrita_stream_t stream) {
  if (!logits || !out || B < 1 || V < 1 || ld < V || sample_size < 1) return QRITA_EINVAL_ARG;
  if (dtype != QRITA_DTYPE_F32 && dtype != QRITA_DTYPE_BF16) return QRITA_EINVAL_ARG;
  const int n = sample_size < V ? sample_size : V;
  const int threads = 128, blocks = (B + threads - 1) / threads;
  if (dtype == QRITA_DTYPE_F32)
    row_stats_kernel<float><<<blocks, threads, 0, (cudaStream_t)stream>>>((const float *)logits, ld, B, n, out);
  else
    row_stats_kernel<uint16_t><<<blocks, threads, 0, (cudaStream_t)stream>>>((const uint16_t *)logits, ld, B, n,
                                                                             out);
  return cudaGetLastError() == cudaSuccess ? QRITA_OK : QRITA_ECUDA;
}

}  // extern "C"
