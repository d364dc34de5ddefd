// qrita_lmhead.cu — SURVEY.md §8(f) rank 3: the LM-head GEMM with the truncation's streaming pass
// fused into its epilogue.
//
// logits[b][v] = sum_k hidden[b][k] * weight[v][k]   (bf16 inputs, fp32 accumulation; the LM head of
// the model whose logits the reference truncates).  The reference has no code for
// this producer; its consumer is the path of qrita_impl.cuh (pipeline.truncate_topk_topp,
// pipeline.py:199-239; oracle.oracle_topk_topp, oracle.py:70-89).
//
// Kernel (sm_100a): one CTA per 128-vocabulary x BN-batch tile.  A = weight tile (128 x 64 bf16,
// K-major, 128-byte swizzle) and B = hidden tile (BN x 64) are brought in by TMA (cp.async.bulk.tensor)
// through a STAGES-deep mbarrier ring; one thread issues tcgen05.mma (M = 128, N = BN, K = 16) into a
// TMEM accumulator; after the last k-block the four warps read their 32 TMEM lanes (= 32 vocabulary
// rows) with tcgen05.ld and run the epilogue.
//
// Fused epilogue (qrita_lmhead_topk_topp): besides writing the logits once, each tile does the work
// of the staged pipeline's streaming pass (qrita_staged.cuh qrita_stream) for its 128 columns of every
// batch row — outliers z >= thr(row) compacted into the row's outlier buffer, row max / min key and
// the first non-finite column folded into the row aggregate.  The sigma plan (thr) comes from the
// first min(4096, V) logits of each row, computed first by the same kernel (same tiles, same k order,
// hence bit-identical values) and planned by qrita_prep.  The row tails (qrita_tail) then resolve from
// the outlier buffers; on a sigma hit the logits are never read back — only rows that miss (or tie at
// a cut inside the row) read their logits row.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "qrita_impl.cuh"
#include "qrita_internal.h"

namespace qrita {
void pw_tree_build(int n, PwTree &t);  // qrita_capi.cu
}

namespace qrita {
namespace lmh {

constexpr int kBM = 128;               // vocabulary rows per tile (MMA M, TMEM lanes)
constexpr int kBK = 64;                // K per stage: one 128-byte swizzle atom of bf16
constexpr int kUK = 16;                // K per tcgen05.mma (kind::f16)
constexpr int kABytes = kBM * kBK * 2; // 16 KB
constexpr int kSample = 4096;          // the sigma plan's sample prefix (sigma_trunc.py:69-82)

struct Args {
  int V, B, d;                   // logits [B, V]
  int vlimit;                    // columns written / streamed: V, or the sample prefix
  float *logits;                 // [B][ld] (row b, column v)
  int64_t ld;
  // fused streaming epilogue (plans == nullptr: plain GEMM)
  const RowPlan *plans;
  RowAgg *agg;
  uint32_t *cand_bits, *cand_idx;
  int xcap;
};

__device__ __forceinline__ uint64_t smem_desc_sw128(const void *p) {
  // SM100 shared-memory matrix descriptor: start >> 4, LBO 16 B (unused for swizzled K-major),
  // SBO 1024 B (8 rows x 128 B), version 1, layout SWIZZLE_128B (cute/arch/mma_sm100_desc.hpp)
  const uint32_t a = smem_u32(p);
  return (uint64_t)((a & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *tm, int c0, int c1,
                                            unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      :: "r"(smem_u32(dst)), "l"((uint64_t)tm), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      :: "r"(tmem_d), "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
}

__device__ __forceinline__ void mma_commit(unsigned long long *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               :: "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <int BN>
constexpr uint32_t tmem_cols() { return BN <= 32 ? 32u : BN <= 64 ? 64u : BN <= 128 ? 128u : 256u; }

template <int BN, int STAGES>
constexpr size_t dyn_smem() { return 1024 + (size_t)STAGES * (kABytes + BN * kBK * 2); }

template <int BN, int STAGES>
__global__ void __launch_bounds__(128, 1) lmh_gemm(const __grid_constant__ CUtensorMap tmW,
                                                   const __grid_constant__ CUtensorMap tmH, Args a) {
  constexpr int kBBytes = BN * kBK * 2;
  constexpr uint32_t kCols = tmem_cols<BN>();
  // instruction descriptor (kind::f16): D f32, A / B bf16, both K-major, N >> 3, M >> 4
  constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                              ((uint32_t)(kBM >> 4) << 24);
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t *sA = smem, *sB = smem + (size_t)STAGES * kABytes;
  __shared__ unsigned long long full[STAGES], empty[STAGES], tfull;
  __shared__ uint32_t tmem_base;
  __shared__ uint32_t s_mx[4][BN], s_mn[4][BN];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int v0 = blockIdx.x * kBM, b0 = blockIdx.y * BN;
  const int nk = a.d / kBK;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1u); mbar_init(&empty[s], 1u); }
    mbar_init(&tfull, 1u);
    mbar_fence_init();
    asm volatile("prefetch.tensormap [%0];" :: "l"((uint64_t)&tmW) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"((uint64_t)&tmH) : "memory");
  }
  if (warp == 1) {  // TMEM: kCols fp32 columns x 128 lanes; the same warp frees them
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(&tmem_base)), "r"(kCols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;

  if (warp == 0 && lane == 0) {
    // TMA producer
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (uint32_t)(kb / STAGES) & 1u;
      if (kb >= STAGES) mbar_wait(&empty[s], ph ^ 1u);
      mbar_arrive_expect_tx(&full[s], (uint32_t)(kABytes + kBBytes));
      tma_load_2d(sA + (size_t)s * kABytes, &tmW, kb * kBK, v0, &full[s]);
      tma_load_2d(sB + (size_t)s * kBBytes, &tmH, kb * kBK, b0, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    // MMA issuer: one thread for the CTA
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (uint32_t)(kb / STAGES) & 1u;
      mbar_wait(&full[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint64_t ad = smem_desc_sw128(sA + (size_t)s * kABytes);
      const uint64_t bd = smem_desc_sw128(sB + (size_t)s * kBBytes);
#pragma unroll
      for (int k = 0; k < kBK / kUK; ++k)  // +32 bytes along K inside the swizzle atom: start += 2
        mma_bf16(tmem, ad + (uint64_t)(2 * k), bd + (uint64_t)(2 * k), kIdesc, (kb | k) ? 1u : 0u);
      mma_commit(&empty[s]);  // the stage is free once these MMAs have read it
    }
    mma_commit(&tfull);       // accumulator complete
  }
  __syncwarp();

  // epilogue: warp w owns TMEM lanes 32w..32w+31 = vocabulary rows v0 + 32w + lane
  mbar_wait(&tfull, 0u);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int v = v0 + warp * 32 + lane;
  const bool vok = v < a.vlimit;
  const bool fused = a.plans != nullptr;
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, r);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int b = b0 + c0 + j;
      if (b >= a.B) break;  // uniform over the warp
      const float z = __uint_as_float(r[j]);
      if (vok && a.logits) a.logits[(size_t)b * a.ld + v] = z;
      if (fused) {
        const RowPlan *pl = a.plans + b;
        const float thr = pl->has_thr ? __uint_as_float(bits_of_key(pl->key_thr)) : __uint_as_float(0x7fffffffu);
        const bool out = vok && z >= thr;  // outlier iff z >= thr (qrita_stream)
        const uint32_t bal = __ballot_sync(0xffffffffu, out);
        if (bal) {
          uint32_t pos = 0u;
          if (lane == 0) pos = atomicAdd(&a.agg[b].count, (uint32_t)__popc(bal));
          pos = __shfl_sync(0xffffffffu, pos, 0) + (uint32_t)__popc(bal & lt);
          if (out && pos < (uint32_t)a.xcap) {
            a.cand_bits[(size_t)b * a.xcap + pos] = __float_as_uint(z);
            a.cand_idx[(size_t)b * a.xcap + pos] = (uint32_t)v;
          }
        }
        const uint32_t key = key_of_bits(__float_as_uint(z));
        if (vok && !(fabsf(z) <= 3.402823466e38f)) atomicMin(&a.agg[b].nf_col, (uint32_t)v);
        const uint32_t mx = warp_max(vok ? key : 0u), mn = warp_min(vok ? key : 0xffffffffu);
        if (lane == 0) { s_mx[warp][c0 + j] = mx; s_mn[warp][c0 + j] = mn; }
      }
    }
  }
  if (fused) {
    __syncthreads();
    for (int c = tid; c < BN && b0 + c < a.B; c += 128) {
      const uint32_t mx = max(max(s_mx[0][c], s_mx[1][c]), max(s_mx[2][c], s_mx[3][c]));
      const uint32_t mn = min(min(s_mn[0][c], s_mn[1][c]), min(s_mn[2][c], s_mn[3][c]));
      atomicMax(&a.agg[b0 + c].maxkey, mx);
      atomicMin(&a.agg[b0 + c].minkey, mn);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(kCols) : "memory");
}

// ---------------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// [rows, d] bf16 row-major (leading dimension ld elements) as a K-major TMA map, box 64 x box_rows
bool make_map(CUtensorMap *tm, const void *base, int rows, int d, int64_t ld, int box_rows) {
  PFN_cuTensorMapEncodeTiled_v12000 fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, int STAGES>
cudaError_t launch_bn(const CUtensorMap &tw, const CUtensorMap &th, const Args &a, int vtiles, cudaStream_t st) {
  static int optin[kMaxDevices] = {};
  int dummy = 0;
  cudaError_t e = per_device_once(optin, [](int, int &v) {
    v = 1;
    return cudaFuncSetAttribute(lmh_gemm<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)dyn_smem<BN, STAGES>());
  }, dummy);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)vtiles, (unsigned)((a.B + BN - 1) / BN));
  lmh_gemm<BN, STAGES><<<grid, 128, dyn_smem<BN, STAGES>(), st>>>(tw, th, a);
  return cudaGetLastError();
}

int batch_tile(int B) {
  if (B <= 16) return 16;
  if (B <= 32) return 32;
  if (B <= 64) return 64;
  if (B <= 128) return 128;
  return 256;
}

// logits (or the sample prefix, a.vlimit columns) for all rows; the fused epilogue when a.plans
int run_gemm(const void *hidden, int64_t ld_h, const void *weight, int64_t ld_w, const Args &a, cudaStream_t st) {
  const int bn = batch_tile(a.B);
  CUtensorMap tw, th;
  if (!make_map(&tw, weight, a.V, a.d, ld_w, kBM) || !make_map(&th, hidden, a.B, a.d, ld_h, bn))
    return QRITA_ECUDA;
  const int vtiles = (a.vlimit + kBM - 1) / kBM;
  cudaError_t e;
  switch (bn) {
    case 16: e = launch_bn<16, 8>(tw, th, a, vtiles, st); break;
    case 32: e = launch_bn<32, 8>(tw, th, a, vtiles, st); break;
    case 64: e = launch_bn<64, 6>(tw, th, a, vtiles, st); break;
    case 128: e = launch_bn<128, 5>(tw, th, a, vtiles, st); break;
    default: e = launch_bn<256, 4>(tw, th, a, vtiles, st); break;
  }
  return e == cudaSuccess ? QRITA_OK : QRITA_ECUDA;
}

int check_shapes(const void *hidden, int64_t ld_h, const void *weight, int64_t ld_w, int B, int V, int d) {
  if (!hidden || !weight || B < 1 || V < 1 || d < kBK || d % kBK) return QRITA_EINVAL_ARG;
  if (ld_h < d || ld_w < d || (ld_h * 2) % 16 || (ld_w * 2) % 16) return QRITA_EINVAL_ARG;
  if (((uintptr_t)hidden & 15u) || ((uintptr_t)weight & 15u)) return QRITA_EINVAL_ARG;
  return QRITA_OK;
}

struct LmhLayout {
  size_t ws, sample, total;
};
LmhLayout lmh_layout(int B, int V) {
  LmhLayout L;
  L.ws = 0;
  size_t off = align_up(ws_layout(B, V).total, 256);
  L.sample = off;
  off = align_up(off + (size_t)B * kSample * 4, 256);
  L.total = off;
  return L;
}

}  // namespace lmh
}  // namespace qrita

using namespace qrita;
using namespace qrita::lmh;

extern "C" {

int qrita_lmhead_logits(const void *hidden, int64_t ld_h, const void *weight, int64_t ld_w, int B, int V, int d,
                        float *logits, int64_t ld_logits, qrita_stream_t stream) {
  int rc = check_shapes(hidden, ld_h, weight, ld_w, B, V, d);
  if (rc != QRITA_OK) return rc;
  if (!logits || ld_logits < V) return QRITA_EINVAL_ARG;
  Args a;
  memset(&a, 0, sizeof(a));
  a.V = V; a.B = B; a.d = d; a.vlimit = V; a.logits = logits; a.ld = ld_logits;
  return run_gemm(hidden, ld_h, weight, ld_w, a, (cudaStream_t)stream);
}

size_t qrita_lmhead_workspace_bytes(int B, int V) {
  if (B < 1 || V < 1) return 0;
  return lmh_layout(B, V).total;
}

int qrita_lmhead_topk_topp(const void *hidden, int64_t ld_h, const void *weight, int64_t ld_w, int B, int V, int d,
                           const int64_t *k, const double *p, float *logits, int64_t ld_logits, int32_t *kept_idx,
                           int64_t ld_idx, int32_t *kept_count, qrita_row_metrics *metrics, void *workspace,
                           size_t ws_bytes, int flags, qrita_stream_t stream) {
  int rc = check_shapes(hidden, ld_h, weight, ld_w, B, V, d);
  if (rc != QRITA_OK) return rc;
  if (!logits || ld_logits < V || !k || !p || !workspace) return QRITA_EINVAL_ARG;
  if (!kept_idx || ld_idx < 1 || (!kept_count && !metrics)) return QRITA_EINVAL_ARG;
  if (flags & ~(QRITA_SEARCH_BINARY | QRITA_NO_SIGMA | QRITA_FORCE_FALLBACK | QRITA_NO_DUP | QRITA_DEBUG_TIMING))
    return QRITA_EINVAL_ARG;
  const LmhLayout LL = lmh_layout(B, V);
  if (ws_bytes < LL.total || ((uintptr_t)workspace & 255u)) return QRITA_EWORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t *ws = (uint8_t *)workspace;
  const WsLayout L = ws_layout(B, V);
  float *sample = (float *)(ws + LL.sample);
  const int ns = V < kSample ? V : kSample;

  // (1) the sample prefix of every row: the same GEMM tiles as the full pass (bit-identical values)
  Args a;
  memset(&a, 0, sizeof(a));
  a.V = V; a.B = B; a.d = d; a.vlimit = ns; a.logits = sample; a.ld = kSample;
  rc = run_gemm(hidden, ld_h, weight, ld_w, a, st);
  if (rc != QRITA_OK) return rc;

  // (2) row plans from the sample (qrita_prep), which also resets the row aggregates
  Params P;
  memset(&P, 0, sizeof(P));
  P.logits = sample; P.ld_in = kSample; P.out = nullptr; P.ld_out = V;
  P.B = B; P.V = V; P.dtype = QRITA_DTYPE_F32; P.flags = flags; P.sample_size = kSample;
  P.k = k; P.p = p; P.kept_count = kept_count; P.metrics = metrics;
  P.kept_idx = kept_idx; P.ld_idx = ld_idx;
  P.plans = (RowPlan *)(ws + L.plans);
  P.agg = (RowAgg *)(ws + L.agg);
  P.handled = (int32_t *)(ws + L.handled);
  P.cand_bits = (uint32_t *)(ws + L.cand_bits);
  P.cand_idx = (uint32_t *)(ws + L.cand_idx);
  P.status = (int32_t *)(ws + L.status);
  P.nf_col = (int32_t *)(ws + L.nf_col);
  P.dbg = (unsigned long long *)(ws + L.dbg);
  P.nchunks = (V + kChunk - 1) / kChunk;
  P.xcap = row_cap(V);
  P.total_items = B * P.nchunks;
  pw_tree_build(ns, P.tree);
  qrita_prep<float><<<B, kThreads, 0, st>>>(P);
  if (cudaGetLastError() != cudaSuccess) return QRITA_ECUDA;

  // (3) the full GEMM with the streaming pass in its epilogue
  a.vlimit = V; a.logits = logits; a.ld = ld_logits;
  a.plans = P.plans; a.agg = P.agg; a.cand_bits = P.cand_bits; a.cand_idx = P.cand_idx; a.xcap = P.xcap;
  rc = run_gemm(hidden, ld_h, weight, ld_w, a, st);
  if (rc != QRITA_OK) return rc;

  // (4) row tails from the outlier buffers; the logits are read only by rows that need the row
  P.logits = logits; P.ld_in = ld_logits;
  static int optin[kMaxDevices] = {};
  int dummy = 0;
  cudaError_t e = per_device_once(optin, [](int, int &v) {
    v = 1;
    return cudaFuncSetAttribute(qrita_tail<float, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTailDynSmem);
  }, dummy);
  if (e != cudaSuccess) return QRITA_ECUDA;
  static int optin1[kMaxDevices] = {};
  e = per_device_once(optin1, [](int, int &v) {
    v = 1;
    return cudaFuncSetAttribute(qrita_tail<float, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTailDynSmem);
  }, dummy);
  if (e != cudaSuccess) return QRITA_ECUDA;
  if (flags & QRITA_SEARCH_BINARY) qrita_tail<float, 1><<<B, kThreads, kTailDynSmem, st>>>(P);
  else qrita_tail<float, 3><<<B, kThreads, kTailDynSmem, st>>>(P);
  return cudaGetLastError() == cudaSuccess ? QRITA_OK : QRITA_ECUDA;
}

}  // extern "C"
