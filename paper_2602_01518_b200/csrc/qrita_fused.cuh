// qrita_fused.cuh — the fused single-kernel pipeline (default).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "qrita_resolve.cuh"

namespace qrita {

// ------------------------------------------------------------------------------------------------
// Fused single-kernel pipeline: one CTA owns one row at a time
// ------------------------------------------------------------------------------------------------
// CTA = 8 warps (kThreads), two CTAs per SM (128 registers each), persistent over rows
// (row = blockIdx.x + i * gridDim.x).  Per row:
//   ring      the row streams through kRing 4 KB shared-memory stages filled by bulk copies
//             (cp.async.bulk, L2 evict_first) that complete on per-stage mbarriers; thread 0 fills the
//             ring at row start, then the warp that consumes chunk c refills its stage with chunk
//             c + kRing (no producer warp, no empty barriers);
//   plan      the sigma plan is computed from the first sample stages in place (plan_begin /
//             plan_sample: the numpy pairwise statistics of sigma_trunc.py:69-103);
//   stream    warp w consumes chunks w, w + 8, ...: row max and NaN-propagating max |x|, outliers
//             (z >= threshold) appended straight into shared memory X with one warp-aggregated slot
//             reservation per chunk and counted into key bins, the -inf (or copy) background written
//             to HBM with streaming 128-bit stores;
//   resolve   tail_resolve on X, with the ring reused as its work area.
// The row never leaves the SM between reading and resolving: no inter-kernel dependency, one launch
// per call; the other CTA on the SM streams while this one resolves.
// Shared memory per CTA (two CTAs per SM, <= 113 KB each): X = kCapXF outliers (44 KB; further ones
// spill to the row's HBM buffer) + a ring of kRing 4 KB stages (60 KB in flight per CTA, 120 KB per
// SM), which doubles as the tail's work area once the row is consumed, + the outliers' key-bin
// histogram (4 KB), counted while streaming.
constexpr int kStageBytes = 4096;
constexpr int kCapXF = 5632;
constexpr int kRing = 15;
#ifndef QRITA_STREAM_HIST  // count the outliers into key bins while streaming (else in the tail, from X)
#define QRITA_STREAM_HIST 1
#endif
#ifndef QRITA_L2_PREFETCH
#define QRITA_L2_PREFETCH 0  // measured neutral on cfg2 / cfg4 (tools/ab2.sh); kept as an option
#endif

constexpr int kFusedThreads = kThreads;  // 8 warps: stream, plan and resolve (no producer warp)
static_assert(kRing >= 8, "ring must hold the sigma sample (<= 6 stages) plus slack");
static_assert(kRing * kStageBytes >= kWorkBytes, "the ring doubles as the tail work area");
static_assert(sizeof(PlanScratch) <= (size_t)kCapXF * 8, "plan scratch aliases the outlier area");

struct FusedSmem {
  TailSmem tail;
  RowPlan pl;
  unsigned long long full[kRing];   // stage filled (TMA transaction bytes)
  uint32_t seq[kRing];              // chunk sequence number last issued into the stage
  uint32_t n_x;                     // outliers of the current row (all of them, even past kCapX)
  uint32_t hist[kNB];               // outliers per key bin (tail_resolve's bin sort)
  uint32_t wmx[kWarps], wnf[kWarps];
};

// Wait until chunk g has landed in its stage.  Warps consume chunks round-robin, so a warp may ask for
// use n of a stage before use n-1 has landed; a bare parity wait would then see the completed phase
// n-2 and return early.  The producer records g in seq[] only after use n-1 was consumed, so once seq
// shows g the barrier is in phase n (copy in flight) or n+1 (landed) and the parity is unambiguous.
__device__ __forceinline__ void stage_wait(FusedSmem &fs, uint32_t g) {
  const uint32_t slot = g % kRing;
  while (ld_relaxed_smem(&fs.seq[slot]) != g) {
  }
  mbar_wait(&fs.full[slot], (g / kRing) & 1u);
}

template <typename T>
__device__ __forceinline__ float elem_f(T v) { return __uint_as_float(Elem<T>::bits(v)); }

__device__ __forceinline__ float max3_nan(float a, float b, float c) {
  float r;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
template <int N> struct MaskT { using type = uint32_t; };
template <> struct MaskT<64> { using type = unsigned long long; };

// One consumer warp, one chunk of CE = 4 KB / sizeof(T) elements staged in shared memory.  Per
// element: a 3-input max (row max), a 3-input NaN-propagating max of |x| (non-finite detection), one
// compare folded into a per-lane outlier bit mask.  Then one warp scan + one shared atomic reserve
// the chunk's slots in X, and each lane copies its outliers (re-read from the stage by bit index).
template <typename T, bool HIST>
__device__ __forceinline__ void consume_chunk(const uint8_t *stage, int c0, int n, float thr, bool write_bg,
                                              bool write_copy, T *dst, uint32_t *n_x, uint32_t *xb,
                                              uint32_t *xi, uint32_t *gxb, uint32_t *gxi, uint32_t gcap,
                                              uint32_t *hist, uint32_t bl, int bsh, float &rmx, float &ramx) {
  using VT = typename Vec<T>::type;
  constexpr int W = Vec<T>::W;
  constexpr int CE = kStageBytes / (int)sizeof(T);
  constexpr int U = CE / (32 * W);
  using M = typename MaskT<U * W>::type;
  const int lane = threadIdx.x & 31;
  const T *st = reinterpret_cast<const T *>(stage);
  M m = 0;
  if (n == CE) {
    const VT *sv = reinterpret_cast<const VT *>(stage);
    VT v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = sv[u * 32 + lane];
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int w = 0; w < W; w += 2) {
        const float x0 = lane_f<T>(v[u], w), x1 = lane_f<T>(v[u], w + 1);
        rmx = max3f(rmx, x0, x1);
        ramx = max3_nan(ramx, fabsf(x0), fabsf(x1));
        m |= (M)(x0 >= thr) << (u * W + w);
        m |= (M)(x1 >= thr) << (u * W + w + 1);
      }
    }
    // one branch per chunk; lane-based pointer with immediate offsets; -inf from one register
    VT *pd = reinterpret_cast<VT *>(dst) + lane;
    if (write_bg) {
      const uint32_t ni = sizeof(T) == 4 ? 0xff800000u : 0xff80ff80u;
#pragma unroll
      for (int u = 0; u < U; ++u) st_cs_splat4(pd + u * 32, ni);
    } else if (write_copy) {
#pragma unroll
      for (int u = 0; u < U; ++u) __stcs(pd + u * 32, v[u]);
    }
  } else {  // ragged tail chunk of the row: element-wise, same (u, lane, w) layout
    for (int u = 0; u < U; ++u) {
      const int e = (u * 32 + lane) * W;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        if (e + w < n) {
          const float x = elem_f<T>(st[e + w]);
          rmx = fmaxf(rmx, x);
          ramx = max_nan(ramx, fabsf(x));
          m |= (M)(x >= thr) << (u * W + w);
          if (write_bg || write_copy) dst[e + w] = write_bg ? Elem<T>::neg_inf() : st[e + w];
        }
      }
    }
  }
  // reserve this warp's outlier slots in X (one shared atomic per chunk)
  const uint32_t cnt = (uint32_t)__popcll((unsigned long long)m);
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  if (total == 0u) return;
  uint32_t base = 0u;
  if (lane == 31) base = atomicAdd(n_x, total);
  base = __shfl_sync(0xffffffffu, base, 31);
  if (base >= (uint32_t)kCapXF + gcap) return;  // X is full: the outliers are only counted
  uint32_t pos = base + incl - cnt;
  const int le = lane * W;  // element of bit j: (j / W) * 32 * W + lane * W + j % W
  while (m) {
    const int j = __ffsll((long long)m) - 1;
    m &= m - 1;
    const int e = ((j & ~(W - 1)) << 5) + le + (j & (W - 1));
    const uint32_t bits = Elem<T>::bits(st[e]);
    if (HIST) {
      // a positive threshold makes every outlier a positive float: its key is bits | 2^31
      const uint32_t key = bl >= 0x80000000u ? (bits | 0x80000000u) : key_of_bits(bits);
      const uint32_t bin = (key - bl - 1u) >> bsh;
      atomicAdd(&hist[bin < (uint32_t)kNB ? bin : (uint32_t)(kNB - 1)], 1u);
    }
    if (pos < (uint32_t)kCapXF) {
      xb[pos] = bits; xi[pos] = (uint32_t)(c0 + e);
    } else if (pos - (uint32_t)kCapXF < gcap) {  // spill past shared memory into the row's HBM buffer
      gxb[pos - kCapXF] = bits; gxi[pos - kCapXF] = (uint32_t)(c0 + e);
    }
    ++pos;
  }
}

template <typename T, int NP>
__global__ void __launch_bounds__(kFusedThreads, 2) qrita_fused(Params P) {
  extern __shared__ __align__(128) uint8_t dsmem[];
  __shared__ FusedSmem fs;
  constexpr int CE = kStageBytes / (int)sizeof(T);
  uint32_t *xb = (uint32_t *)dsmem;
  uint32_t *xi = xb + kCapXF;
  uint8_t *ring = dsmem + (size_t)kCapXF * 8;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int V = P.V;
  const int nch = (V + CE - 1) / CE;
  if (tid == 0) {
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&fs.full[i], 1u);
      fs.seq[i] = 0xffffffffu;
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (P.topp16) pdl_wait();  // qrita_topp16 (the previous kernel) has written `handled`
  const unsigned long long pol = l2_evict_first_policy();
  uint32_t g0 = 0u;  // chunks of this CTA's earlier rows: the ring's stage sequence
  for (int row = blockIdx.x; row < P.B; row += gridDim.x) {
    if (P.topp16 && P.handled[row]) continue;  // finished by qrita_topp16 (launched just before)
    const T *in = (const T *)P.logits + (size_t)row * P.ld_in;
    // chunk c of the row -> stage (g0 + c) % kRing; seq records the chunk before its copy is issued
    auto issue = [&](int c) {
      const uint32_t g = g0 + (uint32_t)c, slot = g % kRing;
      st_relaxed_smem(&fs.seq[slot], g);
      const uint32_t bytes = (uint32_t)(min(CE, V - c * CE) * (int)sizeof(T));
      mbar_arrive_expect_tx(&fs.full[slot], bytes);
      tma_load_1d(ring + (size_t)slot * kStageBytes, in + (size_t)c * CE, bytes, &fs.full[slot], pol);
#if QRITA_L2_PREFETCH
      // the chunk kRing further on goes to L2 now: its ring load then waits for an L2 hit instead of a
      // loaded HBM round trip, doubling the bytes in flight per CTA without shared memory
      if (c + kRing < nch)
        l2_prefetch_bulk(in + (size_t)(c + kRing) * CE, (uint32_t)(min(CE, V - (c + kRing) * CE) * (int)sizeof(T)));
#endif
    };
    if (tid == 0) {  // fill the ring; afterwards each consumed stage is refilled by its consumer
      fence_proxy_async_smem();  // the previous row's tail wrote the ring through the generic proxy
      for (int c = 0; c < kRing && c < nch; ++c) issue(c);
    }
    {
      QRITA_TSTAMP(0);
      if ((P.flags & QRITA_DEBUG_TIMING) && tid == 0) {  // debug: which SM ran the row
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        P.dbg[(size_t)row * 16 + 15] = smid;
      }
      // (1) plan: the sample-independent part while the first stages land, then the sample in place
      if (tid == 32) { fs.n_x = 0u; plan_begin(P, row, &fs.pl); }  // warp 1, while warp 0 fills the ring
      const int ns = P.tree.n_leaves > 0 ? (P.tree.n + CE - 1) / CE : 0;
      for (int i = tid; i < kNB; i += kThreads) fs.hist[i] = 0u;
      for (int j = 0; j < ns; ++j) stage_wait(fs, g0 + (uint32_t)j);
      tsync();
      plan_sample<T>(P, [&](int i) -> float {
        const uint32_t g = g0 + (uint32_t)(i / CE);
        return elem_f<T>(reinterpret_cast<const T *>(ring + (size_t)(g % kRing) * kStageBytes)[i % CE]);
      }, in, *reinterpret_cast<PlanScratch *>(dsmem), &fs.pl);
      tsync();
      QRITA_TSTAMP(1);
      const RowPlan &pl = fs.pl;  // read from shared memory on use (keeps the stream loop's registers free)
      const bool inplace = (P.flags & QRITA_INPLACE) != 0;
      const int mode = pl.mode;
      const float thr = pl.has_thr ? __uint_as_float(bits_of_key(pl.key_thr)) : __uint_as_float(0x7fffffffu);
      const bool hist = QRITA_STREAM_HIST && (mode == MODE_TOPK || mode == MODE_TOPKP);
      const uint32_t bl = pl.key_thr - 1u;
      const int bsh = pl.bsh;
      const bool has_out = P.out != nullptr;  // index-only calls write no masked logits
      const bool write_bg = has_out && !inplace && (mode == MODE_TOPK || mode == MODE_TOPKP || mode == MODE_INVALID);
      const bool write_copy = has_out && !inplace && mode == MODE_PASS;
      T *dst = (T *)P.out + (size_t)row * P.ld_out;
      uint32_t *gxb = P.cand_bits + (size_t)row * P.xcap, *gxi = P.cand_idx + (size_t)row * P.xcap;
      // (2) stream: warp w consumes chunks w, w + 8, ...
      float rmx = -3.402823466e38f, ramx = 0.0f;  // row max; NaN-propagating max |x| (non-finite check)
      for (int c = warp; c < nch; c += kWarps) {
        const uint32_t g = g0 + (uint32_t)c, slot = g % kRing;
        stage_wait(fs, g);
        if (hist)
          consume_chunk<T, true>(ring + (size_t)slot * kStageBytes, c * CE, min(CE, V - c * CE), thr, write_bg,
                                 write_copy, dst + (size_t)c * CE, &fs.n_x, xb, xi, gxb, gxi, (uint32_t)P.xcap,
                                 fs.hist, bl, bsh, rmx, ramx);
        else
          consume_chunk<T, false>(ring + (size_t)slot * kStageBytes, c * CE, min(CE, V - c * CE), thr, write_bg,
                                  write_copy, dst + (size_t)c * CE, &fs.n_x, xb, xi, gxb, gxi, (uint32_t)P.xcap,
                                  fs.hist, bl, bsh, rmx, ramx);
        __syncwarp();
        if (lane == 0 && c + kRing < nch) {  // refill this stage with the chunk kRing ahead
          fence_proxy_async_smem();
          issue(c + kRing);
        }
      }
      {
        const uint32_t mx = warp_max(key_of_bits(__float_as_uint(rmx)));
        const bool nf = __any_sync(0xffffffffu, !(ramx <= 3.402823466e38f));
        if (lane == 0) { fs.wmx[warp] = mx; fs.wnf[warp] = nf ? 0u : 0xffffffffu; }
      }
      tsync();
      QRITA_TSTAMP(2);
      // minkey 0: the full-row fallback searches start below every finite key; a non-finite row
      // reports column 0 and the error path locates the first bad column exactly
      uint32_t maxkey = 0u, minkey = 0u, nf_col = 0xffffffffu;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        maxkey = max(maxkey, fs.wmx[w]);
        nf_col = min(nf_col, fs.wnf[w]);
      }
      // (3) resolve; every stage of this row has been consumed, so the ring is the work area
      tail_resolve<T, NP>(P, row, pl, xb, xi, ring, fs.tail, fs.n_x, false, maxkey, minkey, nf_col,
                          (uint32_t)kCapXF, gxb, gxi, (uint32_t)P.xcap, QRITA_STREAM_HIST ? fs.hist : nullptr, pl.bsh,
                          (size_t)kRing * kStageBytes);
    }
    g0 += (uint32_t)nch;
    __syncthreads();  // row done: the ring and X may be refilled
  }
}

constexpr size_t kFusedDynSmem = (size_t)kCapXF * 8 + (size_t)kRing * kStageBytes;

template <typename T, int NP>
static cudaError_t launch_fused(const Params &P, cudaStream_t st, bool pdl = false) {
  static int grid_caps[kMaxDevices] = {};  // per instantiation and device
  int grid_cap = 0;
  cudaError_t e = per_device_once(grid_caps, [](int dev, int &cap) {
    cudaError_t e = cudaFuncSetAttribute(qrita_fused<T, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kFusedDynSmem);
    if (e != cudaSuccess) return e;
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qrita_fused<T, NP>, kFusedThreads, kFusedDynSmem);
    if (e != cudaSuccess) return e;
    cap = sms * (per_sm < 1 ? 1 : per_sm);
    return cudaSuccess;
  }, grid_cap);
  if (e != cudaSuccess) return e;
  // Balanced persistent grid: every CTA gets the same number of rows (no partial last wave), as
  // long as that keeps >= 3/4 of the CTA slots (and their ring bytes in flight) busy.
  int grid = P.B < grid_cap ? P.B : grid_cap;
  if (P.B > grid_cap && !getenv("QRITA_UNBALANCED")) {
    const int per = (P.B + grid_cap - 1) / grid_cap;
    const int bal = (P.B + per - 1) / per;
    if (4 * bal >= 3 * grid_cap) grid = bal;
  }
  if (!pdl) {
    qrita_fused<T, NP><<<grid, kFusedThreads, kFusedDynSmem, st>>>(P);
    return cudaGetLastError();
  }
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kFusedThreads);
  cfg.dynamicSmemBytes = kFusedDynSmem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, qrita_fused<T, NP>, P);
}

}  // namespace qrita
