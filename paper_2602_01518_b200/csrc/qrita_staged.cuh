// qrita_staged.cuh — the staged pipeline for unaligned rows: qrita_stream and qrita_tail
// (after qrita_prep), chained with programmatic dependent launch.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "qrita_resolve.cuh"

namespace qrita {

// Row tail of the staged pipeline: waits for qrita_stream, gathers the row's outliers from its HBM
// row buffer into shared memory in one round trip, then resolves.
template <typename T, int NP>
__device__ __forceinline__ void tail_body(const Params &P, uint8_t *dsmem, TailSmem &sm) {
  const int row = blockIdx.x;
  pdl_wait();  // outliers and row aggregates of qrita_stream (and plans of qrita_prep)
  QRITA_TSTAMP(0);
  const int tid = threadIdx.x;
  RowPlan pl;
  {
    const uint4 *src4 = reinterpret_cast<const uint4 *>(P.plans + row);
    uint4 *dst4 = reinterpret_cast<uint4 *>(&pl);
#pragma unroll
    for (int i = 0; i < (int)(sizeof(RowPlan) / 16); ++i) dst4[i] = __ldcg(src4 + i);
  }
  uint32_t *xb = (uint32_t *)dsmem;      // [kCapX] outlier bits
  uint32_t *xi = xb + kCapX;             // [kCapX] outlier indices
  // one round trip: the row aggregate, and speculatively the first kSpecTail * kThreads outliers of
  // the row buffer (coalesced; entries past the count are ignored)
  const size_t rb = (size_t)row * P.xcap;
  const uint4 a0 = __ldcg(reinterpret_cast<const uint4 *>(P.agg + row));
  const uint4 a1 = __ldcg(reinterpret_cast<const uint4 *>(P.agg + row) + 1);
  uint32_t vb[kSpecTail], vi[kSpecTail];
#pragma unroll
  for (int j = 0; j < kSpecTail; ++j) {
    const int i = tid + j * kThreads;
    vb[j] = vi[j] = 0u;
    if (i < P.xcap) { vb[j] = __ldcg(P.cand_bits + rb + i); vi[j] = __ldcg(P.cand_idx + rb + i); }
  }
  const uint32_t n_c = a0.x;
  const bool overflow = a1.x != 0u || n_c > (uint32_t)P.xcap;
  if (pl.has_thr && !overflow && n_c <= (uint32_t)kCapX) {
#pragma unroll
    for (int j = 0; j < kSpecTail; ++j) {
      const uint32_t i = (uint32_t)(tid + j * kThreads);
      if (i < n_c) { xb[i] = vb[j]; xi[i] = vi[j]; }
    }
    for (uint32_t i0 = kSpecTail * kThreads; i0 < n_c; i0 += 4 * kThreads) {
      uint32_t b4[4], x4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t i = i0 + tid + j * kThreads;
        b4[j] = x4[j] = 0u;
        if (i < n_c) { b4[j] = __ldcg(P.cand_bits + rb + i); x4[j] = __ldcg(P.cand_idx + rb + i); }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t i = i0 + tid + j * kThreads;
        if (i < n_c) { xb[i] = b4[j]; xi[i] = x4[j]; }
      }
    }
  }
  tsync();
  QRITA_TSTAMP(1);
  tail_resolve<T, NP>(P, row, pl, xb, xi, dsmem + (size_t)kCapX * 8, sm, n_c, overflow, a0.y, a0.z, a0.w,
                      (uint32_t)kCapX);
}

template <typename T, int NP>
__global__ void __launch_bounds__(kThreads, 2) qrita_tail(Params P) {
  extern __shared__ __align__(16) uint8_t dsmem[];
  __shared__ TailSmem sm;
  tail_body<T, NP>(P, dsmem, sm);
}

// ------------------------------------------------------------------------------------------------
// K1: streaming pass + row tails
// ------------------------------------------------------------------------------------------------
// One warp streams one 1024-element chunk: 128-bit loads (8 per lane for fp32, 4 for bf16), chunk
// max / min with NaN-propagating min/max (non-finite values surface in the chunk extrema, no
// per-element test), order-stable outlier compaction with ballot/popc staged in shared memory and
// written out coalesced, and the output background (-inf for top-k rows, a copy for passthrough
// rows).  No block barriers: warps never wait for each other.
template <typename T, bool VEC>
__global__ void __launch_bounds__(kStreamThreads, 3) qrita_stream(Params P) {
  using VT = typename Vec<T>::type;
  constexpr int W = Vec<T>::W;
  constexpr int U = kChunk / (32 * W);
  constexpr int NWB = kStreamThreads / 32;
  static_assert(U * 32 * W == kChunk, "chunk shape");
  __shared__ uint32_t s_cb[NWB][kCapChunk];
  __shared__ uint32_t s_ci[NWB][kCapChunk];
  pdl_launch_dependents();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gwarp = (int)((blockIdx.x * kStreamThreads + threadIdx.x) >> 5);
  const int nwarps = (int)((gridDim.x * kStreamThreads) >> 5);
  const int nch = P.nchunks;
  const bool inplace = (P.flags & QRITA_INPLACE) != 0;
  const uint32_t lt = (1u << lane) - 1u;
  const float qnan = __uint_as_float(0x7fffffffu);
  const unsigned long long keep_pol = l2_evict_last_policy();
  bool waited = false;

  for (int item = gwarp; item < P.total_items; item += nwarps) {
    const int row = item / nch, c = item - row * nch;
    const int c0 = c * kChunk;
    const int n = min(kChunk, P.V - c0);
    const bool whole = VEC && n == kChunk;  // warp-uniform fast path
    const T *src = (const T *)P.logits + (size_t)row * P.ld_in + c0;
    T *dst = (T *)P.out + (size_t)row * P.ld_out + c0;
    VT v[U];
    if (whole) {
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldcs(reinterpret_cast<const VT *>(src + (u * 32 + lane) * W));
    }
    if (!waited) {  // the logits never depend on qrita_prep; the plans do
      pdl_wait();
      waited = true;
    }
    const RowPlan *plp = P.plans + row;
    const int mode = plp->mode;
    // outlier iff z >= thr (float compare: -0.0 == +0.0 as in the reference); NaN threshold = none
    const float thr = plp->has_thr ? __uint_as_float(bits_of_key(plp->key_thr)) : qnan;
    const bool has_out = P.out != nullptr;  // index-only calls write no masked logits
    const bool write_bg = has_out && !inplace && (mode == MODE_TOPK || mode == MODE_TOPKP || mode == MODE_INVALID);
    const bool write_copy = has_out && !inplace && mode == MODE_PASS;
    // finite identities, so lanes without elements (ragged chunks) never look non-finite
    float fmx = -3.402823466e38f, fmn = 3.402823466e38f;
    uint32_t base = 0u;
    if (whole) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = (u * 32 + lane) * W;
        uint32_t bal[W];
        uint32_t any = 0u;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const float x = lane_f<T>(v[u], w);
          fmx = max_nan(fmx, x);
          fmn = min_nan(fmn, x);
          bal[w] = __ballot_sync(0xffffffffu, x >= thr);
          any |= bal[w];
        }
        if (any) {  // warp-uniform: stage this slot's outliers in index order (u, lane, w)
          uint32_t q = base;
#pragma unroll
          for (int w = 0; w < W; ++w) q += (uint32_t)__popc(bal[w] & lt);
#pragma unroll
          for (int w = 0; w < W; ++w) {
            if ((bal[w] >> lane) & 1u) {
              if (q < (uint32_t)kCapChunk) {
                s_cb[wib][q] = lane_bits<T>(v[u], w);
                s_ci[wib][q] = (uint32_t)(c0 + e + w);
              }
              ++q;
            }
          }
#pragma unroll
          for (int w = 0; w < W; ++w) base += (uint32_t)__popc(bal[w]);
        }
        if (write_bg) __stcs(reinterpret_cast<VT *>(dst + e), neg_inf_vec<T>());
        else if (write_copy) __stcs(reinterpret_cast<VT *>(dst + e), v[u]);
      }
    } else {
      // ragged / unaligned chunk: element-wise, same (u, lane, w) order
      for (int u = 0; u < U; ++u) {
        const int e = (u * 32 + lane) * W;
        uint32_t bal[W];
        uint32_t b[W];
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const bool valid = e + w < n;
          b[w] = valid ? Elem<T>::bits(src[e + w]) : 0u;
          const float x = __uint_as_float(b[w]);
          if (valid) {
            fmx = max_nan(fmx, x);
            fmn = min_nan(fmn, x);
          }
          bal[w] = __ballot_sync(0xffffffffu, valid && x >= thr);
          if (valid && (write_bg || write_copy)) dst[e + w] = write_bg ? Elem<T>::neg_inf() : src[e + w];
        }
        uint32_t q = base;
#pragma unroll
        for (int w = 0; w < W; ++w) q += (uint32_t)__popc(bal[w] & lt);
#pragma unroll
        for (int w = 0; w < W; ++w) {
          if ((bal[w] >> lane) & 1u) {
            if (q < (uint32_t)kCapChunk) { s_cb[wib][q] = b[w]; s_ci[wib][q] = (uint32_t)(c0 + e + w); }
            ++q;
          }
          base += (uint32_t)__popc(bal[w]);
        }
      }
    }
    // chunk statistics; NaN / inf anywhere shows up in the NaN-propagating extrema
    const bool nf_lane = f_nonfinite(fmx) || f_nonfinite(fmn);
    const uint32_t nf = __any_sync(0xffffffffu, nf_lane) ? (uint32_t)c0 : 0xffffffffu;
    const uint32_t mx = warp_max(key_of_bits(__float_as_uint(fmx)));
    const uint32_t mn = warp_min(key_of_bits(__float_as_uint(fmn)));
    __syncwarp();
    // fold the chunk into the row aggregate; reserve room in the row's outlier buffer
    RowAgg *ag = P.agg + row;
    uint32_t pos = 0u;
    if (lane == 0) {
      if (base) pos = atomicAdd(&ag->count, base);
      atomicMax(&ag->maxkey, mx);
      atomicMin(&ag->minkey, mn);
      if (nf != 0xffffffffu) atomicMin(&ag->nf_col, nf);
      if (base > (uint32_t)kCapChunk) atomicOr(&ag->ovf, 1u);
    }
    pos = __shfl_sync(0xffffffffu, pos, 0);
    const uint32_t nst = base < (uint32_t)kCapChunk ? base : (uint32_t)kCapChunk;
    const size_t rb = (size_t)row * P.xcap;
    // outliers are re-read by the row tail: keep them in L2 (evict_last) while the logits stream
    // past with evict_first
    for (uint32_t j = lane; j < nst && pos + j < (uint32_t)P.xcap; j += 32) {
      st_keep_u32(P.cand_bits + rb + pos + j, s_cb[wib][j], keep_pol);
      st_keep_u32(P.cand_idx + rb + pos + j, s_ci[wib][j], keep_pol);
    }
    __syncwarp();
  }
  if (!waited) pdl_wait();
}

constexpr size_t kTailDynSmem = (size_t)kCapX * 8 + (size_t)kWorkBytes;

template <typename T, int NP, bool VEC>
static cudaError_t launch_pipeline(const Params &P, cudaStream_t st, cudaEvent_t prep_done,
                                   cudaEvent_t stream_done) {
  static int stream_grids[kMaxDevices] = {};  // per instantiation and device
  int stream_grid = 0;
  cudaError_t e0 = per_device_once(stream_grids, [](int dev, int &grid) {
    cudaError_t e = cudaFuncSetAttribute(qrita_tail<T, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kTailDynSmem);
    if (e != cudaSuccess) return e;
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qrita_stream<T, VEC>, kStreamThreads, 0);
    if (e != cudaSuccess) return e;
    // two streaming CTAs per SM leave room for one row-tail CTA, so tails run while rows stream
    int want = 3;
    if (const char *ev = getenv("QRITA_STREAM_CTAS_PER_SM")) want = atoi(ev);
    if (want < 1) want = 1;
    grid = sms * (per_sm < want ? (per_sm < 1 ? 1 : per_sm) : want);
    return cudaSuccess;
  }, stream_grid);
  if (e0 != cudaSuccess) return e0;
  const Params &PP = P;
  qrita_prep<T><<<P.B, 256, 0, st>>>(PP);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (prep_done) {
    e = cudaEventRecord(prep_done, st);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = prep_done ? 0 : 1;  // exact timing when profiled
  cudaLaunchConfig_t cfg = {};
  const int warps_needed = P.total_items;
  int grid = (warps_needed + kStreamThreads / 32 - 1) / (kStreamThreads / 32);
  if (grid > stream_grid) grid = stream_grid;
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kStreamThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, qrita_stream<T, VEC>, PP);
  if (e != cudaSuccess) return e;
  if (stream_done) {
    e = cudaEventRecord(stream_done, st);
    if (e != cudaSuccess) return e;
  }
  attr[0].val.programmaticStreamSerializationAllowed = stream_done ? 0 : 1;
  cfg.gridDim = dim3((unsigned)P.B);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kTailDynSmem;
  return cudaLaunchKernelEx(&cfg, qrita_tail<T, NP>, PP);
}

}  // namespace qrita
