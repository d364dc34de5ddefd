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
#include <stdlib.h>
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
  // in-kernel sample and plans (plan_rows, one batch tile): the nst sample vocabulary tiles come first
  // (all in the first round of the persistent grid); then every CTA plans its share of the rows
  int plan_rows, nst;
  uint32_t *done, *ready;        // [batch tiles] sample tiles written / rows planned
};

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// tile t -> (vocabulary tile, batch tile); with in-kernel plans the sample tiles come first
__device__ __forceinline__ void tile_of(const Args &a, int t, int vt, int bt, int &vx, int &y, bool &sample) {
  sample = false;
  if (!a.plan_rows) { vx = t % vt; y = t / vt; return; }
  const int ns = a.nst * bt;
  if (t < ns) { vx = t % a.nst; y = t / a.nst; sample = true; return; }
  const int r = t - ns, w = vt - a.nst;
  vx = a.nst + r % w;
  y = r / w;
}

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
constexpr uint32_t tmem_cols() { return BN <= 16 ? 32u : BN <= 32 ? 64u : BN <= 64 ? 128u : BN <= 128 ? 256u : 512u; }

template <int BN, int STAGES>
constexpr size_t dyn_smem() { return 1024 + (size_t)STAGES * (kABytes + BN * kBK * 2); }

// order key of fp32 bits (qrita_device.cuh key_of_bits), branch-free: -0.0 ranks as +0.0
__device__ __forceinline__ uint32_t lmh_key(uint32_t b) {
  b = b == 0x80000000u ? 0u : b;
  return b ^ ((uint32_t)((int32_t)b >> 31) | 0x80000000u);
}

constexpr int kEpiWarps = 8;
constexpr int kMaxPlanRows = 4;                 // rows per CTA whose plan_begin runs up front                    // two per TMEM lane quarter, each half of the columns
constexpr int kGemmThreads = 64 + 32 * kEpiWarps;

__device__ __forceinline__ void epi_sync() {    // the epilogue warps only
  asm volatile("barrier.sync 1, %0;" :: "n"(32 * kEpiWarps) : "memory");
}

// Persistent, warp-specialised: warp 0 = TMA producer, warp 1 = MMA issuer (and TMEM owner), warps
// 2..9 = epilogue.  Two TMEM accumulators (2 x BN columns): the epilogue of tile i overlaps the MMAs
// of tile i + 1.  Tiles: t = blockIdx.x + i * gridDim.x over (vocab tile, batch tile), vocab fastest.
template <int BN, int STAGES>
__global__ void __launch_bounds__(kGemmThreads, 1) lmh_gemm(const __grid_constant__ CUtensorMap tmW,
                                                            const __grid_constant__ CUtensorMap tmH, Args a,
                                                            const __grid_constant__ Params P) {
  constexpr int kBBytes = BN * kBK * 2;
  constexpr uint32_t kCols = tmem_cols<BN>();
  // instruction descriptor (kind::f16): D f32, A / B bf16, both K-major, N >> 3, M >> 4
  constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                              ((uint32_t)(kBM >> 4) << 24);
  constexpr int kHalf = BN / 2;  // columns per epilogue warp
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t *sA = smem, *sB = smem + (size_t)STAGES * kABytes;
  __shared__ unsigned long long full[STAGES], empty[STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  __shared__ uint32_t s_mx[4][BN], s_cnt[4][BN];
  __shared__ __align__(16) float s_thr[BN];
  __shared__ PlanScratch s_sc;
  __shared__ RowPlan s_pls[kMaxPlanRows];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nk = a.d / kBK;
  const int vt = (a.vlimit + kBM - 1) / kBM, bt = (a.B + BN - 1) / BN;
  const int ntiles = vt * bt;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1u); mbar_init(&empty[s], 1u); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1u); mbar_init(&tempty[s], (uint32_t)kEpiWarps); }
    mbar_fence_init();
    asm volatile("prefetch.tensormap [%0];" :: "l"((uint64_t)&tmW) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"((uint64_t)&tmH) : "memory");
  }
  if (warp == 1) {  // TMEM: 2 x BN fp32 columns x 128 lanes; the same warp frees them
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(&tmem_base)), "r"(kCols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  pdl_launch_dependents();  // the row tails may be scheduled (they wait for this grid's results)

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      int g = 0;  // k-blocks issued so far (ring position)
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int vx, y;
        bool smp;
        tile_of(a, t, vt, bt, vx, y, smp);
        const int v0 = vx * kBM, b0 = y * BN;
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % STAGES;
          const uint32_t ph = (uint32_t)(g / STAGES) & 1u;
          if (g >= STAGES) mbar_wait(&empty[s], ph ^ 1u);
          mbar_arrive_expect_tx(&full[s], (uint32_t)(kABytes + kBBytes));
          tma_load_2d(sA + (size_t)s * kABytes, &tmW, kb * kBK, v0, &full[s]);
          tma_load_2d(sB + (size_t)s * kBBytes, &tmH, kb * kBK, b0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer: one thread for the CTA
      int g = 0, i = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int acc = i & 1;
        if (i >= 2) mbar_wait(&tempty[acc], (uint32_t)((i >> 1) - 1) & 1u);  // epilogue drained it
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d_tmem = tmem + (uint32_t)(acc * BN);
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % STAGES;
          const uint32_t ph = (uint32_t)(g / STAGES) & 1u;
          mbar_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t ad = smem_desc_sw128(sA + (size_t)s * kABytes);
          const uint64_t bd = smem_desc_sw128(sB + (size_t)s * kBBytes);
#pragma unroll
          for (int k = 0; k < kBK / kUK; ++k)  // +32 bytes along K inside the swizzle atom: start += 2
            mma_bf16(d_tmem, ad + (uint64_t)(2 * k), bd + (uint64_t)(2 * k), kIdesc, (kb | k) ? 1u : 0u);
          mma_commit(&empty[s]);  // the stage is free once these MMAs have read it
        }
        mma_commit(&tfull[acc]);  // accumulator complete
      }
    }
  } else {
    // epilogue: warp w reads TMEM lane quarter q = w % 4 (vocabulary rows v0 + 32q + lane) and the
    // columns [h * BN/2, (h + 1) * BN/2) of the accumulator
    const int q = warp & 3, h = (warp - 2) >> 2, et = tid - 64;
    const bool fused = a.plans != nullptr;
    const uint32_t lt = (1u << lane) - 1u;
    int i = 0;
    uint32_t planned = 0u;  // batch tiles whose row plans this CTA has seen published
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      int vx, y;
      bool smp;
      tile_of(a, t, vt, bt, vx, y, smp);
      const int v0 = vx * kBM, b0 = y * BN;
      const int acc = i & 1;
      const int v = v0 + q * 32 + lane;
      const bool vok = v < a.vlimit;
      const int nrow = min(BN, a.B - b0);  // rows of the batch tile
      if (a.plan_rows) {
        if (smp) {
          // the sample columns' logits first; once the batch tile's nst sample tiles are written,
          // this CTA plans rows b0 + vx, b0 + vx + nst, ... (qrita_prep's work) and publishes them
          mbar_wait(&tfull[acc], (uint32_t)(i >> 1) & 1u);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t trow0 = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + h * kHalf);
#pragma unroll 1
          for (int c0 = 0; c0 < kHalf; c0 += 16) {
            uint32_t r[16];
            tmem_ld16(trow0 + (uint32_t)c0, r);
            const int cb = h * kHalf + c0, nb = min(16, a.B - (b0 + cb));
            if (vok) {
              float *dst = a.logits + (size_t)(b0 + cb) * a.ld + v;
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (j < nb) dst[(size_t)j * a.ld] = __uint_as_float(r[j]);
            }
          }
          __threadfence();
          epi_sync();
          if (et == 0) atomicAdd(&a.done[y], 1u);
        }
        if (i == 0) {
          // every CTA plans rows blockIdx.x, blockIdx.x + gridDim.x, ... (qrita_prep's work): the
          // sample-independent part for all of them at once (one thread per row), the sample part
          // once the nst sample tiles are written (one batch tile: every CTA's first tile is in it)
          const int myrows = (a.B - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
          for (int r = et; r < myrows && r < kMaxPlanRows; r += 32 * kEpiWarps)
            plan_begin(P, (int)blockIdx.x + r * (int)gridDim.x, &s_pls[r]);
          if (et == 0)
            while (ld_acquire_gpu(&a.done[0]) < (uint32_t)a.nst) __nanosleep(64);
          epi_sync();
          uint32_t np = 0u;
          for (int row = blockIdx.x; row < a.B; row += gridDim.x, ++np) {
            RowPlan &pl = s_pls[np < (uint32_t)kMaxPlanRows ? np : 0];
            const float *lr = a.logits + (size_t)row * a.ld;
            // the default sample (4096 = 32 leaves of 128): thread (leaf L, accumulator j) loads its
            // 16 values at once and runs numpy's leaf loop in registers (plan_sample's order exactly)
            const bool perfect = P.tree.n == 4096 && P.tree.n_leaves == 32;
            if (perfect) {
              const int L = et >> 3, j = et & 7;
              float xv[16];
#pragma unroll
              for (int m = 0; m < 16; ++m) xv[m] = __ldcg(lr + 128 * L + j + 8 * m);
              double r0 = (double)xv[0];
              double r1 = __dmul_rn(r0, r0);
#pragma unroll
              for (int m = 1; m < 16; ++m) {
                const double x = (double)xv[m];
                r0 = __dadd_rn(r0, x);
                r1 = __dadd_rn(r1, __dmul_rn(x, x));
              }
              s_sc.acc[0][L][j] = r0;
              s_sc.acc[1][L][j] = r1;
            }
            if (np >= (uint32_t)kMaxPlanRows && et == 0) plan_begin(P, row, &pl);
            epi_sync();
            plan_sample<float>(P, [&](int ii) -> float { return __ldcg(lr + ii); }, lr, s_sc, &pl, 64, perfect);
            epi_sync();
            if (et == 0) {
              P.plans[row] = pl;
              uint4 *ag = reinterpret_cast<uint4 *>(P.agg + row);
              ag[0] = make_uint4(0u, 0u, 0u, 0xffffffffu);  // count, maxkey, minkey 0 (fused kernel's), nf_col
              ag[1] = make_uint4(0u, 0u, 0u, 0u);
            }
            epi_sync();
          }
          __threadfence();
          epi_sync();
          if (et == 0 && np) atomicAdd(&a.ready[0], np);
        }
        if (!((planned >> (y & 31)) & 1u)) {
          if (et == 0)
            while (ld_acquire_gpu(&a.ready[y]) < (uint32_t)nrow) __nanosleep(64);
          epi_sync();
          planned |= 1u << (y & 31);
        }
      }
      if (fused) {
        for (int c = et; c < BN; c += 32 * kEpiWarps) {  // thresholds of the tile's rows
          const int b = b0 + c;
          float tv = __uint_as_float(0x7fffffffu);  // NaN: no threshold, no outliers
          if (b < a.B && a.plans[b].has_thr) tv = __uint_as_float(bits_of_key(a.plans[b].key_thr));
          s_thr[c] = tv;
        }
        epi_sync();
      }
      mbar_wait(&tfull[acc], (uint32_t)(i >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + h * kHalf);
      // (A) logits; per (quarter, row): outlier count, max key, first non-finite column
#pragma unroll 1
      for (int c0 = 0; c0 < kHalf; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(trow + (uint32_t)c0, r);
        const int cb = h * kHalf + c0;  // first accumulator column of the chunk
        const int nb = min(16, a.B - (b0 + cb));  // rows of the chunk inside the batch (uniform)
        if (a.logits && vok && !smp) {
          float *dst = a.logits + (size_t)(b0 + cb) * a.ld + v;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < nb) dst[(size_t)j * a.ld] = __uint_as_float(r[j]);
        }
        if (fused) {
          float th[16];
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            const float4 t4 = *reinterpret_cast<const float4 *>(&s_thr[cb + j]);
            th[j] = t4.x; th[j + 1] = t4.y; th[j + 2] = t4.z; th[j + 3] = t4.w;
          }
          uint32_t bad = 0u, cnt = 0u, mxs = 0u;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float z = __uint_as_float(r[j]);
            const uint32_t bal = __ballot_sync(0xffffffffu, vok && z >= th[j]);
            bad |= (vok && !(fabsf(z) <= 3.402823466e38f)) ? (1u << j) : 0u;
            const uint32_t mx = warp_max(vok ? lmh_key(r[j]) : 0u);
            if (lane == j) { cnt = (uint32_t)__popc(bal); mxs = mx; }
          }
          if (lane < nb) { s_cnt[q][cb + lane] = cnt; s_mx[q][cb + lane] = mxs; }
          if (__any_sync(0xffffffffu, bad != 0u)) {  // non-finite logits: the first column per row
            for (int j = 0; j < nb; ++j)
              if ((bad >> j) & 1u) atomicMin(&a.agg[b0 + cb + j].nf_col, (uint32_t)v);
          }
        }
      }
      if (!fused) {  // accumulator drained
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        if (lane == 0) mbar_arrive(&tempty[acc]);
        continue;
      }
      // (B) one reservation per (tile, row) in the row's outlier buffer; the row maximum
      epi_sync();
      for (int c = et; c < BN && b0 + c < a.B; c += 32 * kEpiWarps) {
        const int b = b0 + c;
        uint32_t n[4], tot = 0u;
#pragma unroll
        for (int w = 0; w < 4; ++w) { n[w] = s_cnt[w][c]; tot += n[w]; }
        uint32_t base = tot ? atomicAdd(&a.agg[b].count, tot) : 0u;
#pragma unroll
        for (int w = 0; w < 4; ++w) { s_cnt[w][c] = base; base += n[w]; }
        atomicMax(&a.agg[b].maxkey, max(max(s_mx[0][c], s_mx[1][c]), max(s_mx[2][c], s_mx[3][c])));
        // min key 0 (as the fused kernel): full-row fallback searches start below every finite key
        if (v0 == 0 && !a.plan_rows) a.agg[b].minkey = 0u;
      }
      epi_sync();
      // (C) the outliers, from TMEM again, at their reserved positions
#pragma unroll 1
      for (int c0 = 0; c0 < kHalf; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(trow + (uint32_t)c0, r);
        const int cb = h * kHalf + c0;
        const int nb = min(16, a.B - (b0 + cb));
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const bool out = vok && j < nb && __uint_as_float(r[j]) >= s_thr[cb + j];
          const uint32_t bal = __ballot_sync(0xffffffffu, out);
          if (out) {
            const uint32_t pos = s_cnt[q][cb + j] + (uint32_t)__popc(bal & lt);
            if (pos < (uint32_t)a.xcap) {
              const size_t o = (size_t)(b0 + cb + j) * a.xcap + pos;
              a.cand_bits[o] = r[j];
              a.cand_idx[o] = (uint32_t)v;
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      if (lane == 0) mbar_arrive(&tempty[acc]);
      epi_sync();  // s_cnt / s_thr are rewritten for the next tile
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

int sm_count() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

template <int BN, int STAGES>
cudaError_t launch_bn(const CUtensorMap &tw, const CUtensorMap &th, const Args &a, const Params &P, int vtiles,
                      cudaStream_t st) {
  static int optin[kMaxDevices] = {};
  int dummy = 0;
  cudaError_t e = per_device_once(optin, [](int, int &v) {
    v = 1;
    return cudaFuncSetAttribute(lmh_gemm<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)dyn_smem<BN, STAGES>());
  }, dummy);
  if (e != cudaSuccess) return e;
  const int sms = sm_count();
  const int ntiles = vtiles * ((a.B + BN - 1) / BN);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // in-kernel plans: CTAs wait for each other
  attr[0].val.cooperative = a.plan_rows ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ntiles < sms ? ntiles : sms));
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = dyn_smem<BN, STAGES>();
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, lmh_gemm<BN, STAGES>, tw, th, a, P);
}

int batch_tile(int B) {
  if (B <= 16) return 16;
  if (B <= 32) return 32;
  if (B <= 64) return 64;
  if (B <= 128) return 128;
  return 256;
}

// logits (or the sample prefix, a.vlimit columns) for all rows; the fused epilogue when a.plans
int run_gemm(const void *hidden, int64_t ld_h, const void *weight, int64_t ld_w, const Args &a, const Params &P,
             cudaStream_t st) {
  const int bn = batch_tile(a.B);
  CUtensorMap tw, th;
  if (!make_map(&tw, weight, a.V, a.d, ld_w, kBM) || !make_map(&th, hidden, a.B, a.d, ld_h, bn))
    return QRITA_ECUDA;
  const int vtiles = (a.vlimit + kBM - 1) / kBM;
  cudaError_t e;
  switch (bn) {
    case 16: e = launch_bn<16, 8>(tw, th, a, P, vtiles, st); break;
    case 32: e = launch_bn<32, 8>(tw, th, a, P, vtiles, st); break;
    case 64: e = launch_bn<64, 6>(tw, th, a, P, vtiles, st); break;
    case 128: e = launch_bn<128, 5>(tw, th, a, P, vtiles, st); break;
    default: e = launch_bn<256, 4>(tw, th, a, P, vtiles, st); break;
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
  size_t ws, sample, counters, total;
};
LmhLayout lmh_layout(int B, int V) {
  LmhLayout L;
  L.ws = 0;
  size_t off = align_up(ws_layout(B, V).total, 256);
  L.sample = off;
  off = align_up(off + (size_t)B * kSample * 4, 256);
  L.counters = off;
  off = align_up(off + 2 * 4 * (size_t)(B + 15) / 16 + 256, 256);
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
  Params P;
  memset(&P, 0, sizeof(P));
  return run_gemm(hidden, ld_h, weight, ld_w, a, P, (cudaStream_t)stream);
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

  Params P;
  memset(&P, 0, sizeof(P));
  P.logits = logits; P.ld_in = ld_logits; P.out = nullptr; P.ld_out = V;
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

  Args a;
  memset(&a, 0, sizeof(a));
  a.V = V; a.B = B; a.d = d; a.vlimit = V; a.logits = logits; a.ld = ld_logits;
  a.plans = P.plans; a.agg = P.agg; a.cand_bits = P.cand_bits; a.cand_idx = P.cand_idx; a.xcap = P.xcap;
  const int bn = batch_tile(B), bt = (B + bn - 1) / bn, nst = (ns + kBM - 1) / kBM;
  const int vt = (V + kBM - 1) / kBM;
  const int grid = vt * bt < sm_count() ? vt * bt : sm_count();
  bool one_launch = bt == 1 && nst <= grid && !(getenv("QRITA_LMH_PREP"));
  if (one_launch) {
    // one launch: the sample tiles come first, their CTAs plan the rows, every epilogue waits for
    // its batch tile's plans (the MMAs of the next tile run meanwhile)
    uint32_t *cnt = (uint32_t *)(ws + LL.counters);
    if (cudaMemsetAsync(cnt, 0, 2 * 4 * (size_t)bt, st) != cudaSuccess) return QRITA_ECUDA;
    Args a1 = a;
    a1.plan_rows = 1; a1.nst = nst; a1.done = cnt; a1.ready = cnt + bt;
    if (run_gemm(hidden, ld_h, weight, ld_w, a1, P, st) != QRITA_OK) {
      // the cooperative launch needs every CTA resident at once (an MPS share of the SMs may not
      // allow it): take the three-launch path instead
      (void)cudaGetLastError();
      one_launch = false;
    }
  }
  if (!one_launch) {
    // (1) the sample prefix of every row: the same GEMM tiles as the full pass (bit-identical values)
    Args as = a;
    as.plans = nullptr; as.vlimit = ns; as.logits = sample; as.ld = kSample;
    Params P0;
    memset(&P0, 0, sizeof(P0));
    rc = run_gemm(hidden, ld_h, weight, ld_w, as, P0, st);
    if (rc != QRITA_OK) return rc;
    // (2) row plans from the sample (qrita_prep), which also resets the row aggregates
    Params PS = P;
    PS.logits = sample; PS.ld_in = kSample;
    qrita_prep<float><<<B, kThreads, 0, st>>>(PS);
    if (cudaGetLastError() != cudaSuccess) return QRITA_ECUDA;
    // (3) the full GEMM with the streaming pass in its epilogue
    rc = run_gemm(hidden, ld_h, weight, ld_w, a, P, st);
    if (rc != QRITA_OK) return rc;
  }

  // (4) row tails from the outlier buffers; the logits are read only by rows that need the row
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
  // programmatic dependent launch: the tail CTAs take the SMs the GEMM's last round leaves idle and
  // wait there (griddepcontrol.wait in qrita_tail) for the GEMM's results
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)B);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kTailDynSmem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = (flags & QRITA_SEARCH_BINARY) ? cudaLaunchKernelEx(&cfg, qrita_tail<float, 1>, (const Params)P)
                                    : cudaLaunchKernelEx(&cfg, qrita_tail<float, 3>, (const Params)P);
  return e == cudaSuccess ? QRITA_OK : QRITA_ECUDA;
}

}  // extern "C"
