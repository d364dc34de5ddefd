// qrita_impl.cuh — B200 (sm_100a) exact Top-k / Top-p truncation kernels.
//
// Reference path (arxiv/paper_2602_01518, pkg/src/sigmatop):
//   engine.run_batch (engine.py:82-113) -> pipeline.truncate_topk_topp (pipeline.py:199-239)
//     -> sigma_trunc.{row_stats, lookup_delta_*, threshold_from, gather_outliers, is_hit}
//        (sigma_trunc.py:69-138)
//     -> pivot_search.{quaternary,binary}_{topk,topp} (pivot_search.py:93-244)
//     -> pipeline.finalize_mask / _apply_plan (pipeline.py:47-78)
// Ground truth: oracle.oracle_topk_topp (oracle.py:70-89).
//
// Two pipelines behind one C entry point (DESIGN.md has the full story):
//   qrita_fused  (default; rows 16-byte aligned) one launch, one CTA owns one row at a time, two
//                CTAs per SM, persistent over rows.  The row streams once through a ring of 4 KB
//                shared-memory stages filled by bulk copies (cp.async.bulk + mbarrier); the sigma plan
//                is computed in place from the first stages; outliers are compacted straight into
//                shared memory while the -inf / copy background is written; the row tail (bin-sort
//                resolve, or the pivot searches / distinct-value path on the rare full-row cases)
//                runs in the same CTA on the same shared memory.
//   staged       (unaligned rows, or QRITA_STAGED) qrita_prep -> qrita_stream -> qrita_tail chained
//                with programmatic dependent launch; outliers go through per-row HBM buffers.
// Both share tail_resolve and compute bit-identical results.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "qrita_types.cuh"

namespace qrita {

// The two 200-entry quantile tables (tables.py:13-57) — numeric data, required for
// the sigma threshold to equal the reference's.
static __constant__ double c_topk_table[kTableSize] = {
     2.576,  2.319,  2.178,  2.064,  1.968,  1.892,  1.819,  1.757,  1.708,  1.659,
     1.616,  1.568,  1.526,  1.492,  1.456,  1.420,  1.382,  1.342,  1.309,  1.280,
     1.249,  1.221,  1.193,  1.169,  1.145,  1.121,  1.095,  1.073,  1.050,  1.030,
     1.008,  0.987,  0.966,  0.945,  0.926,  0.910,  0.891,  0.871,  0.854,  0.837,
     0.819,  0.803,  0.784,  0.767,  0.753,  0.734,  0.719,  0.702,  0.690,  0.675,
     0.658,  0.640,  0.625,  0.609,  0.595,  0.578,  0.564,  0.550,  0.537,  0.521,
     0.509,  0.495,  0.481,  0.466,  0.453,  0.439,  0.424,  0.410,  0.397,  0.383,
     0.370,  0.356,  0.343,  0.330,  0.316,  0.302,  0.289,  0.274,  0.261,  0.247,
     0.235,  0.223,  0.209,  0.196,  0.184,  0.172,  0.159,  0.149,  0.137,  0.124,
     0.112,  0.100,  0.086,  0.074,  0.062,  0.050,  0.035,  0.023,  0.009, -0.003,
    -0.015, -0.027, -0.039, -0.052, -0.063, -0.074, -0.085, -0.097, -0.109, -0.122,
    -0.134, -0.147, -0.158, -0.171, -0.184, -0.196, -0.210, -0.223, -0.235, -0.248,
    -0.261, -0.275, -0.289, -0.302, -0.317, -0.328, -0.341, -0.353, -0.368, -0.382,
    -0.396, -0.410, -0.426, -0.439, -0.452, -0.465, -0.480, -0.493, -0.507, -0.521,
    -0.537, -0.551, -0.568, -0.582, -0.597, -0.614, -0.628, -0.643, -0.658, -0.673,
    -0.691, -0.706, -0.721, -0.738, -0.754, -0.769, -0.789, -0.808, -0.824, -0.838,
    -0.857, -0.877, -0.893, -0.912, -0.929, -0.947, -0.965, -0.983, -1.003, -1.027,
    -1.050, -1.070, -1.092, -1.117, -1.139, -1.162, -1.189, -1.216, -1.241, -1.272,
    -1.300, -1.330, -1.367, -1.404, -1.441, -1.485, -1.523, -1.564, -1.607, -1.658,
    -1.710, -1.778, -1.832, -1.901, -1.978, -2.068, -2.174, -2.325, -2.577, -3.813,
};
static __constant__ double c_topp_table[kTableSize] = {
     3.656,  3.650,  3.650,  3.650,  3.626,  3.626,  3.626,  3.514,  3.514,  3.503,
     3.503,  3.434,  3.434,  3.428,  3.428,  3.387,  3.380,  3.380,  3.376,  3.373,
     3.373,  3.356,  3.354,  3.354,  3.291,  3.249,  3.234,  3.214,  3.198,  3.198,
     3.185,  3.177,  3.177,  3.165,  3.164,  3.161,  3.138,  3.120,  3.115,  3.113,
     3.093,  3.066,  3.054,  3.043,  3.037,  3.023,  2.993,  2.991,  2.976,  2.970,
     2.952,  2.946,  2.932,  2.908,  2.902,  2.895,  2.886,  2.874,  2.861,  2.844,
     2.836,  2.810,  2.801,  2.790,  2.784,  2.779,  2.767,  2.757,  2.745,  2.733,
     2.723,  2.716,  2.693,  2.678,  2.671,  2.656,  2.649,  2.629,  2.611,  2.595,
     2.592,  2.585,  2.574,  2.550,  2.543,  2.534,  2.521,  2.518,  2.497,  2.485,
     2.468,  2.450,  2.441,  2.430,  2.412,  2.402,  2.389,  2.383,  2.377,  2.364,
     2.349,  2.338,  2.332,  2.319,  2.310,  2.301,  2.282,  2.274,  2.266,  2.250,
     2.242,  2.236,  2.226,  2.215,  2.207,  2.196,  2.179,  2.171,  2.162,  2.147,
     2.135,  2.121,  2.109,  2.095,  2.085,  2.073,  2.063,  2.045,  2.030,  2.016,
     2.003,  1.992,  1.983,  1.972,  1.960,  1.949,  1.940,  1.928,  1.912,  1.897,
     1.881,  1.869,  1.854,  1.838,  1.824,  1.807,  1.792,  1.779,  1.764,  1.751,
     1.739,  1.726,  1.711,  1.697,  1.685,  1.668,  1.652,  1.636,  1.622,  1.603,
     1.585,  1.568,  1.551,  1.534,  1.513,  1.499,  1.480,  1.464,  1.441,  1.422,
     1.394,  1.373,  1.347,  1.320,  1.296,  1.270,  1.246,  1.219,  1.190,  1.163,
     1.135,  1.104,  1.073,  1.041,  1.006,  0.969,  0.931,  0.894,  0.851,  0.806,
     0.757,  0.702,  0.643,  0.574,  0.498,  0.405,  0.288,  0.134, -0.110, -3.813,
};

// ------------------------------------------------------------------------------------------------
// Element access
// ------------------------------------------------------------------------------------------------
template <typename T> struct Elem;
template <> struct Elem<float> {
  static __device__ __forceinline__ uint32_t bits(float v) { return __float_as_uint(v); }
  static __device__ __forceinline__ float neg_inf() { return __uint_as_float(0xff800000u); }
  static __device__ __forceinline__ float from_bits(uint32_t b) { return __uint_as_float(b); }
};
template <> struct Elem<uint16_t> {  // bf16 carried as raw bits; upcast to fp32 is exact
  static __device__ __forceinline__ uint32_t bits(uint16_t v) { return ((uint32_t)v) << 16; }
  static __device__ __forceinline__ uint16_t neg_inf() { return (uint16_t)0xff80u; }
  static __device__ __forceinline__ uint16_t from_bits(uint32_t b) { return (uint16_t)(b >> 16); }
};

// 128-bit vectors of a dtype and their lanes as fp32 bit patterns
template <typename T> struct Vec;
template <> struct Vec<float> { using type = float4; static constexpr int W = 4; };
template <> struct Vec<uint16_t> { using type = uint4; static constexpr int W = 8; };

template <typename T>
__device__ __forceinline__ uint32_t lane_bits(const typename Vec<T>::type &v, int w);
template <>
__device__ __forceinline__ uint32_t lane_bits<float>(const float4 &v, int w) {
  return __float_as_uint(w == 0 ? v.x : w == 1 ? v.y : w == 2 ? v.z : v.w);
}
template <>
__device__ __forceinline__ uint32_t lane_bits<uint16_t>(const uint4 &v, int w) {
  const uint32_t x = (w >> 1) == 0 ? v.x : (w >> 1) == 1 ? v.y : (w >> 1) == 2 ? v.z : v.w;
  return (w & 1) ? (x & 0xffff0000u) : (x << 16);
}

template <typename T>
__device__ __forceinline__ typename Vec<T>::type neg_inf_vec();
template <> __device__ __forceinline__ float4 neg_inf_vec<float>() {
  const float n = __uint_as_float(0xff800000u);
  return make_float4(n, n, n, n);
}
template <> __device__ __forceinline__ uint4 neg_inf_vec<uint16_t>() {
  return make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u);
}

// Per-element comparison of a 128-bit vector against the logit whose order key is K, as bit masks
// (bit w = element w): value order == key order for finite logits, and IEEE equality already treats
// -0.0 == +0.0, so full-row passes compare values directly instead of converting every element to a
// key (fp32 compares; packed bf16x2 compares for bf16).
template <typename T> struct VecCmp;
template <> struct VecCmp<float> {
  float kv;
  __device__ __forceinline__ explicit VecCmp(uint32_t K) { kv = __uint_as_float(bits_of_key(K)); }
  __device__ __forceinline__ void masks(const float4 &v, uint32_t &gt, uint32_t &eq) const {
    gt = (v.x > kv ? 1u : 0u) | (v.y > kv ? 2u : 0u) | (v.z > kv ? 4u : 0u) | (v.w > kv ? 8u : 0u);
    eq = (v.x == kv ? 1u : 0u) | (v.y == kv ? 2u : 0u) | (v.z == kv ? 4u : 0u) | (v.w == kv ? 8u : 0u);
  }
};
template <> struct VecCmp<uint16_t> {
  __nv_bfloat162 k2;
  __device__ __forceinline__ explicit VecCmp(uint32_t K) {
    const uint32_t kb = bits_of_key(K) >> 16;
    const uint32_t w = kb | (kb << 16);
    k2 = *reinterpret_cast<const __nv_bfloat162 *>(&w);
  }
  __device__ __forceinline__ void masks(const uint4 &v, uint32_t &gt, uint32_t &eq) const {
    const uint32_t wd[4] = {v.x, v.y, v.z, v.w};
    gt = eq = 0u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __nv_bfloat162 x = *reinterpret_cast<const __nv_bfloat162 *>(&wd[i]);
      const uint32_t g = __hgt2_mask(x, k2), e = __heq2_mask(x, k2);
      gt |= ((g & 1u) | ((g >> 15) & 2u)) << (2 * i);
      eq |= ((e & 1u) | ((e >> 15) & 2u)) << (2 * i);
    }
  }
};

// ------------------------------------------------------------------------------------------------
// K0: per-row preparation (sigma_trunc.py:69-103; mode routing of pipeline.py:199-218)
// ------------------------------------------------------------------------------------------------
// One leaf of numpy's pairwise summation (n <= 128): 8 accumulators, then the remainder.
template <typename T, bool SQUARE>
__device__ double leaf_sum(const T *a, int n) {
  auto val = [&](int i) -> double {
    const double x = (double)__uint_as_float(Elem<T>::bits(a[i]));
    return SQUARE ? __dmul_rn(x, x) : x;
  };
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, val(i));
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = val(j);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], val(i + j));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, val(i));
  return res;
}

// Post-order evaluation of numpy's pairwise tree over n elements:
//   pw(a, n) = leaf(a, n)                           if n <= 128
//            = pw(a, n2) + pw(a + n2, n - n2)       n2 = n/2 rounded down to a multiple of 8
// Leaves are visited left to right.  Started from the additive identity, this is bit-identical to
// ndarray.sum on a contiguous float64 vector (verified against numpy 2.3 in tests/).
template <class LeafFn>
__device__ double pairwise_tree(int n, LeafFn leaf) {
  int st_off[48], st_n[48], st_state[48];
  double st_left[48];
  int sp = 1;
  st_off[0] = 0; st_n[0] = n; st_state[0] = 0;
  double ret = 0.0;
  bool have = false;
  for (;;) {
    if (!have) {
      const int t = sp - 1;
      if (st_n[t] <= 128) {
        ret = leaf(st_off[t], st_n[t]);
        --sp;
        have = true;
      } else {
        int n2 = st_n[t] / 2;
        n2 -= n2 % 8;
        st_state[t] = 1;
        st_off[sp] = st_off[t]; st_n[sp] = n2; st_state[sp] = 0; ++sp;
      }
    } else {
      if (sp == 0) return ret;
      const int t = sp - 1;
      if (st_state[t] == 1) {
        st_left[t] = ret;
        st_state[t] = 2;
        int n2 = st_n[t] / 2;
        n2 -= n2 % 8;
        st_off[sp] = st_off[t] + n2; st_n[sp] = st_n[t] - n2; st_state[sp] = 0; ++sp;
        have = false;
      } else {
        ret = __dadd_rn(st_left[t], ret);
        --sp;
      }
    }
  }
}

// Serial replay of the pairwise sums straight from global memory (non-default sample sizes only);
// out of line, so its explicit stack stays out of the hot kernels' frames.
template <typename T, bool SQUARE>
__device__ __noinline__ double pairwise_serial(const T *a, int n) {
  return pairwise_tree(n, [&](int o, int m) -> double { return leaf_sum<T, SQUARE>(a + o, m); });
}

// Smallest s with w <= kNB * 2^s: key bins (l, l + 2^s], (l + 2^s, l + 2^(s+1)], ... cover (l, l + w].
__device__ __forceinline__ int bin_shift(uint32_t w) {
  if (w <= (uint32_t)kNB) return 0;
  return (32 - __clz(w - 1u)) - kLogNB;
}

// Debug phase timestamps of the row tail (QRITA_DEBUG_TIMING): P.dbg[row][i] = %globaltimer.
__device__ __forceinline__ void tail_stamp(const Params &P, int row, int i) {
  if ((P.flags & QRITA_DEBUG_TIMING) && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    P.dbg[(size_t)row * 16 + i] = t;
  }
}
#define QRITA_TSTAMP(i) tail_stamp(P, row, (i))

// Row routing (pipeline.py:199-218): which stages run for (k, p).
__device__ __forceinline__ int row_mode(int64_t k, double p, int V) {
  const bool bad_k = !(k >= 1 && k <= (int64_t)V);
  const bool bad_p = !(p > 0.0 && p <= 1.0);
  if (bad_k || bad_p) return MODE_INVALID;
  if (k == V && p == 1.0) return MODE_PASS;
  if (k == V) return MODE_TOPP;
  if (p == 1.0) return MODE_TOPK;
  return MODE_TOPKP;
}

// Scratch of the sigma statistics (shared memory, >= 20 KB).
struct PlanScratch {
  double acc[2][kPwMaxLeaves][8];
  double val[2][2 * kPwMaxLeaves];
  double res[2];
};

// Per-row plan (sigma_trunc.py:69-103; mode routing of pipeline.py:199-218), in two steps so the
// sample-independent part overlaps the sample's arrival:
//   plan_begin (thread 0): mode, table delta (sigma_trunc.py:85-103), exact fixed-point nucleus
//                          thresholds, status word; writes *out (key_thr / mu / sigma / t pending);
//   plan_sample (tail thread group, kThreads threads, tsync barriers): numpy's pairwise mean and mean
//                          square of the sample (bit-replica), sigma, threshold key.  xs(i) returns
//                          sample element i from shared memory; `a` is the row in global memory
//                          (serial fallback for long samples).  Reads *out after a barrier.
__device__ __forceinline__ void plan_begin(const Params &P, int row, RowPlan *out) {
  const int V = P.V;
  const int64_t k = P.k[row];
  const double p = P.p[row];
  const int mode = row_mode(k, p, V);
  const bool want_thr = (mode == MODE_TOPK || mode == MODE_TOPP || mode == MODE_TOPKP) &&
                        !(P.flags & QRITA_NO_SIGMA);
  RowPlan pl;
  pl.key_thr = 0xffffffffu;
  pl.mode = mode;
  pl.k = k;
  pl.p = p;
  pl.mu = pl.sigma = pl.t = 0.0;
  double delta = 0.0;
  if (want_thr) {  // table lookup (sigma_trunc.py:85-96); delta parked in t until plan_sample
    if (mode == MODE_TOPP) {
      int idx = (int)__dmul_rn(p, (double)kTableSize);
      delta = c_topp_table[min(idx, kTableSize - 1)];
    } else {
      int idx = (int)__dmul_rn(__ddiv_rn((double)k, (double)V), (double)kTableSize);
      delta = c_topk_table[min(idx, kTableSize - 1)];
    }
  }
  pl.t = delta;
  if (mode == MODE_TOPP || mode == MODE_TOPKP) {
    pl.t_p = fx_round_threshold(p);
    pl.t_sp = fx_round_threshold(nextafter(p, 2.0));
  } else {
    pl.t_p = fx_zero();
    pl.t_sp = fx_zero();
  }
  pl.has_thr = want_thr ? 1 : 0;
  pl.bsh = 0;
  pl.pad[0] = pl.pad[1] = 0;
  *out = pl;
  const bool bad_k = !(k >= 1 && k <= (int64_t)V);
  const bool bad_p = !(p > 0.0 && p <= 1.0);
  P.status[row] = (bad_k ? ST_BAD_K : 0) | (bad_p ? ST_BAD_P : 0);
  P.nf_col[row] = -1;
}

template <typename T, class SampleAt>
__device__ void plan_sample(const Params &P, SampleAt xs, const T *a, PlanScratch &sc, RowPlan *out) {
  const int tid = threadIdx.x;
  if (!out->has_thr) return;  // uniform per group (written before the caller's barrier)
  const PwTree &tr = P.tree;
  const int n = tr.n;
  const int nl = tr.n_leaves;
  if (nl > 0) {
    // numpy's 8-accumulator leaf loop, one thread per (leaf, accumulator)
    for (int q = tid; q < nl * 8; q += kThreads) {
      const int L = q >> 3, j = q & 7;
      const int o = tr.leaf_off[L], m = tr.leaf_len[L];
      if (m >= 8) {
        double r0 = (double)xs(o + j);
        double r1 = __dmul_rn(r0, r0);
        for (int i = 8; i < m - (m % 8); i += 8) {
          const double x = (double)xs(o + i + j);
          r0 = __dadd_rn(r0, x);
          r1 = __dadd_rn(r1, __dmul_rn(x, x));
        }
        sc.acc[0][L][j] = r0;
        sc.acc[1][L][j] = r1;
      }
    }
    tsync();
    if (n == 4096 && nl == 32) {
      // the default sample is a perfect tree: 32 leaves of 128 combined pairwise level by level
      // (node = left + right), so one warp per sum finishes it with shuffles and no block barriers
      if (tid < 64) {
        const int sq = tid >> 5, L = tid & 31;
        const double *r = sc.acc[sq][L];
        double v = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                             __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double u = __shfl_down_sync(0xffffffffu, v, o);
          if ((L & (2 * o - 1)) == 0) v = __dadd_rn(v, u);
        }
        if (L == 0) sc.res[sq] = v;
      }
      tsync();
      goto finish;
    }
    for (int q = tid; q < nl * 2; q += kThreads) {
      const int L = q >> 1, sq = q & 1;
      const int o = tr.leaf_off[L], m = tr.leaf_len[L];
      double res;
      int i;
      if (m < 8) {
        res = 0.0;
        i = 0;
      } else {
        const double *r = sc.acc[sq][L];
        res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                        __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        i = m - (m % 8);
      }
      for (; i < m; ++i) {
        const double x = (double)xs(o + i);
        res = __dadd_rn(res, sq ? __dmul_rn(x, x) : x);
      }
      sc.val[sq][L] = res;
    }
    tsync();
    // internal nodes level by level: pw(a, n) = pw(a, n2) + pw(a + n2, n - n2)
    int lo = 0;
    for (int h = 0; h < tr.n_levels; ++h) {
      const int hi = tr.level_end[h];
      for (int q = lo + (tid >> 1); q < hi; q += kThreads >> 1) {
        const int sq = tid & 1;
        sc.val[sq][nl + q] = __dadd_rn(sc.val[sq][tr.left[q]], sc.val[sq][tr.right[q]]);
      }
      lo = hi;
      tsync();
    }
    if (tid < 2) sc.res[tid] = sc.val[tid][nl + tr.n_internal - 1 < nl ? 0 : nl + tr.n_internal - 1];
  } else if (tid < 2) {  // long samples (non-default sample_size): serial replay from global
    sc.res[tid] = tid == 0
        ? pairwise_serial<T, false>(a, n) : pairwise_serial<T, true>(a, n);
  }
  tsync();
finish:
  if (tid == 0) {
    const double sum = sc.res[0], sq = sc.res[1];
    // sigma_trunc.py:78-81 — mean, E[x^2] - mu^2 floored at 0, sqrt; no FMA contraction anywhere.
    const double mu = __ddiv_rn(sum, (double)n);
    const double e2 = __ddiv_rn(sq, (double)n);
    const double var = __dsub_rn(e2, __dmul_rn(mu, mu));
    const double sigma = __dsqrt_rn(var > 0.0 ? var : 0.0);
    // safety margin (sigma_trunc.py:99-103)
    const double delta = out->t;
    const double delta_adj = __dsub_rn(delta, __dmul_rn(0.2, fabs(delta)));
    const double t = __dadd_rn(mu, __dmul_rn(delta_adj, sigma));
    // outlier iff float64(z) > t  <=>  z >= f where f is the smallest float above t
    float f = __double2float_rd(t);
    if (!((double)f > t)) f = nextafterf(f, __uint_as_float(0x7f800000u));
    out->key_thr = key_of_bits(__float_as_uint(f));
    // provisional outlier range (t, mu + 6 sigma] for bins counted while streaming; keys above it
    // fall into the last (open) bin, so the binning stays monotone whatever the row holds
    uint32_t khi = key_of_bits(__float_as_uint((float)__dadd_rn(mu, __dmul_rn(6.0, sigma))));
    if (khi < out->key_thr) khi = out->key_thr;
    out->bsh = bin_shift(khi - (out->key_thr - 1u));
    out->mu = mu;
    out->sigma = sigma;
    out->t = t;
  }
}

// K0 of the staged pipeline: one CTA per row stages the sample prefix and writes the row's plan and
// initialises its streaming aggregate.
template <typename T>
__global__ void __launch_bounds__(kThreads) qrita_prep(Params P) {
  __shared__ float s_x[kPwStage];
  __shared__ PlanScratch sc;
  __shared__ RowPlan s_pl;
  pdl_launch_dependents();  // the streaming kernel may start loading logits right away
  const int row = blockIdx.x;
  const int tid = threadIdx.x;
  const T *a = (const T *)P.logits + (size_t)row * P.ld_in;
  const int n = P.tree.n;
  if (P.tree.n_leaves > 0) {
    // batch the loads: 8 independent loads in flight per thread instead of one load per trip
    constexpr int R = 8;
    for (int i0 = tid; i0 < n; i0 += kThreads * R) {
      float tmp[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = i0 + r * kThreads;
        tmp[r] = i < n ? __uint_as_float(Elem<T>::bits(__ldg(a + i))) : 0.0f;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = i0 + r * kThreads;
        if (i < n) s_x[i] = tmp[r];
      }
    }
  }
  if (tid == 0) plan_begin(P, row, &s_pl);
  tsync();
  plan_sample<T>(P, [&](int i) -> float { return s_x[i]; }, a, sc, &s_pl);
  tsync();
  if (tid == 0) {
    P.plans[row] = s_pl;
    uint4 *ag = reinterpret_cast<uint4 *>(P.agg + row);
    ag[0] = make_uint4(0u, 0u, 0xffffffffu, 0xffffffffu);  // count, maxkey, minkey, nf_col
    ag[1] = make_uint4(0u, 0u, 0u, 0u);                     // ovf, done
  }
}

// ------------------------------------------------------------------------------------------------
// Row tail: search + masking, executed by one whole CTA
// ------------------------------------------------------------------------------------------------
// Pivot-search state, owned by warp 0 and broadcast through shared memory.
struct SearchState {
  uint32_t l, r, cl, cr;
  uint32_t done, K, n_gt, n_eq;
  int iters, compact;
  uint32_t n_act, pad;
  Fx Ml, Mr, H;
};

struct TailSmem {
  uint32_t red[2][kWarps][48];  // double-buffered per-warp partials of the block reductions
  uint32_t sel[kWarps];         // per-warp counts of select_nth_eq
  uint32_t u[8];                // broadcast scalars
  uint32_t ctot[kWarps];        // bracket pass: per-warp count totals
  Fx mtot[kWarps];              // bracket pass: per-warp mass totals
  uint32_t scan_u[kWarps];      // bin sort: warp totals of the bin-start scan
  Fx scan_f[2][kWarps];         // bin sort: warp totals of the two mass scans
  uint32_t bstar, nabove, bail, L;
  uint32_t nd, dabort, dK, dngt, dneq, dkmin, dkmax;  // distinct-value top-p
  uint32_t scan_u2[kWarps];
  Fx dH, dMx;
  SearchState st;
};

// ------------------------------------------------------------------------------------------------
// Block scans (one value per thread, thread order); each buffer is reused only after a barrier
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t block_exscan_u32(uint32_t v, uint32_t *buf, uint32_t &total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) buf[warp] = incl;
  tsync();
  uint32_t before = 0u, tot = 0u;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const uint32_t t = buf[w];
    before += (w < warp) ? t : 0u;
    tot += t;
  }
  total = tot;
  return before + incl - v;
}

__device__ __forceinline__ Fx block_exscan_fx(const Fx &v, Fx *buf, Fx &total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Fx incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Fx u;
    u.w0 = __shfl_up_sync(0xffffffffu, incl.w0, o);
    u.w1 = __shfl_up_sync(0xffffffffu, incl.w1, o);
    u.w2 = __shfl_up_sync(0xffffffffu, incl.w2, o);
    if (lane >= o) incl = fx_add(incl, u);
  }
  if (lane == 31) buf[warp] = incl;
  tsync();
  Fx before = fx_zero(), tot = fx_zero();
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const Fx t = buf[w];
    if (w < warp) before = fx_add(before, t);
    tot = fx_add(tot, t);
  }
  total = tot;
  return fx_sub(fx_add(before, incl), v);
}



constexpr int kBins = 256;  // buckets of the bracketing pass (== kThreads: one bucket per thread)

// Block-reduction context.  `par` is block-uniform: consecutive reductions alternate between the
// two partial buffers, so each reduction needs a single barrier.
struct Red {
  TailSmem &sm;
  int par;
  uint32_t *act_key;  // active-set buffer of the pivot searches (keys)
  double *act_pi;     // and, for the top-p search, their probabilities
  int act_cap_k, act_cap_p;
  uint32_t *hcnt;              // [kBins] bracket-pass counts   (aliases the active-set region)
  unsigned long long *hms;     // [5][kBins] bracket-pass masses as 32-bit pieces
  __device__ explicit Red(TailSmem &s) : sm(s), par(0), act_key(nullptr), act_pi(nullptr),
                                         act_cap_k(0), act_cap_p(0), hcnt(nullptr), hms(nullptr) {}
};

// Warp-aggregated slot reservation in a shared counter.
__device__ __forceinline__ uint32_t warp_reserve(uint32_t *ctr, bool want) {
  const uint32_t bal = __ballot_sync(0xffffffffu, want);
  const int lane = threadIdx.x & 31;
  uint32_t base = 0u;
  if (lane == 0 && bal) base = atomicAdd(ctr, (uint32_t)__popc(bal));
  base = __shfl_sync(0xffffffffu, base, 0);
  return base + (uint32_t)__popc(bal & ((1u << lane) - 1u));
}

// Element sources: i -> (fp32 bits, index)
struct SrcX {  // outliers staged in shared memory (index order)
  const uint32_t *bits;
  const uint32_t *idx;
  int n;
  __device__ __forceinline__ void get(int i, uint32_t &b, uint32_t &ix) const { b = bits[i]; ix = idx[i]; }
};
template <typename T>
struct SrcRow {  // the full row in global memory
  const T *row;
  int n;
  __device__ __forceinline__ void get(int i, uint32_t &b, uint32_t &ix) const {
    b = Elem<T>::bits(row[i]);
    ix = (uint32_t)i;
  }
};

// Batched element visits: kLd loads in flight per thread before any is used, so passes over the
// row in global memory are bandwidth- rather than latency-bound.  for_elems calls fn(i, bits, idx)
// for i = tid, tid + kThreads, ... < n.  for_elems_warp keeps whole warps converged (for warp-
// aggregated slot reservation): fn(i, valid, bits, idx) is called by every lane.
constexpr int kLd = 4;
template <class Src, class Fn>
__device__ __forceinline__ void for_elems(const Src &src, int n, Fn fn) {
  for (int i0 = threadIdx.x; i0 < n; i0 += kThreads * kLd) {
    uint32_t b[kLd], x[kLd];
#pragma unroll
    for (int j = 0; j < kLd; ++j) {
      const int i = i0 + j * kThreads;
      b[j] = x[j] = 0u;
      if (i < n) src.get(i, b[j], x[j]);
    }
#pragma unroll
    for (int j = 0; j < kLd; ++j) {
      const int i = i0 + j * kThreads;
      if (i < n) fn(i, b[j], x[j]);
    }
  }
}
template <class Src, class Fn>
__device__ __forceinline__ void for_elems_warp(const Src &src, int n, Fn fn) {
  for (int i0 = threadIdx.x; i0 - (int)threadIdx.x < n; i0 += kThreads * kLd) {
    uint32_t b[kLd], x[kLd];
#pragma unroll
    for (int j = 0; j < kLd; ++j) {
      const int i = i0 + j * kThreads;
      b[j] = x[j] = 0u;
      if (i < n) src.get(i, b[j], x[j]);
    }
#pragma unroll
    for (int j = 0; j < kLd; ++j) {
      const int i = i0 + j * kThreads;
      fn(i, i < n, b[j], x[j]);
    }
  }
}

// Pivot-pass statistics.  Bucket j holds keys in (piv[j], piv[j+1]], piv[NP] = +inf; keys <= piv[0]
// are ignored.  Per bucket: count, min key, count of the min key, exact mass.
template <int NP, bool MASS>
struct Buckets {
  uint32_t cnt[NP], mn[NP], mc[NP];
  Fx ms[MASS ? NP : 1];
};

template <int NP, bool MASS>
__device__ __forceinline__ void bk_init(Buckets<NP, MASS> &b) {
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    b.cnt[j] = 0u; b.mn[j] = 0xffffffffu; b.mc[j] = 0u;
    if (MASS) b.ms[j] = fx_zero();
  }
}

template <int NP, bool MASS>
__device__ __forceinline__ void bk_add(Buckets<NP, MASS> &b, const uint32_t *piv, uint32_t key, const Fx &f) {
  int nb = 0;
#pragma unroll
  for (int j = 0; j < NP; ++j) nb += (key > piv[j]) ? 1 : 0;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    if (nb == j + 1) {
      b.cnt[j] += 1u;
      if (key < b.mn[j]) { b.mn[j] = key; b.mc[j] = 1u; }
      else if (key == b.mn[j]) { b.mc[j] += 1u; }
      if (MASS) b.ms[j] = fx_add(b.ms[j], f);
    }
  }
}

// Block reduction in place: on return every thread holds the block totals in `b`.
// Warp stage with redux.sync, one barrier, then every warp reduces the 16 warp partials itself.
template <int NP, bool MASS>
__device__ void bk_reduce(Buckets<NP, MASS> &b, Red &R) {
  constexpr int NV = 3 * NP + (MASS ? 12 * NP : 0);
  static_assert(NV <= 48, "reduction scratch too small");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t(*red)[48] = R.sm.red[R.par];
  R.par ^= 1;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const uint32_t c = warp_sum(b.cnt[j]);
    const uint32_t m = warp_min(b.mn[j]);
    const uint32_t mc = warp_sum(b.mn[j] == m ? b.mc[j] : 0u);
    if (lane == 0) { red[warp][j] = c; red[warp][NP + j] = m; red[warp][2 * NP + j] = mc; }
    if (MASS) {
      uint32_t q[12];
      fx_split(b.ms[j], q);
#pragma unroll
      for (int i = 0; i < 12; ++i) {
        const uint32_t sum = warp_sum(q[i]);
        if (lane == 0) red[warp][3 * NP + 12 * j + i] = sum;
      }
    }
  }
  tsync();
  const bool act = lane < kWarps;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    b.cnt[j] = warp_sum(act ? red[lane][j] : 0u);
    const uint32_t mv = act ? red[lane][NP + j] : 0xffffffffu;
    const uint32_t m = warp_min(mv);
    b.mn[j] = m;
    b.mc[j] = warp_sum((act && mv == m) ? red[lane][2 * NP + j] : 0u);
    if (MASS) {
      uint32_t q[12];
#pragma unroll
      for (int i = 0; i < 12; ++i) q[i] = warp_sum(act ? red[lane][3 * NP + 12 * j + i] : 0u);
      b.ms[j] = fx_join(q);
    }
  }
}

template <int NP>
__device__ __forceinline__ void make_pivots(uint32_t l, uint32_t r, uint32_t *piv) {
  const unsigned long long w = (unsigned long long)(r - l);
#pragma unroll
  for (int j = 0; j < NP; ++j) piv[j] = l + (uint32_t)((w * (unsigned long long)(j + 1)) / (NP + 1));
}

struct KRes {
  uint32_t K;      // k-th largest key
  uint32_t n_gt;   // keys strictly above K
  uint32_t n_eq;   // keys equal to K
  int iters;
};

// Warp stage of a pivot pass: lane 0 of every warp stores the warp's bucket partials.
template <int NP, bool MASS>
__device__ __forceinline__ void bk_warp_partials(const Buckets<NP, MASS> &b, uint32_t (*red)[48]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const uint32_t c = warp_sum(b.cnt[j]);
    const uint32_t m = warp_min(b.mn[j]);
    const uint32_t mc = warp_sum(b.mn[j] == m ? b.mc[j] : 0u);
    if (lane == 0) { red[warp][j] = c; red[warp][NP + j] = m; red[warp][2 * NP + j] = mc; }
    if (MASS) {
      uint32_t q[12];
      fx_split(b.ms[j], q);
#pragma unroll
      for (int i = 0; i < 12; ++i) {
        const uint32_t sum = warp_sum(q[i]);
        if (lane == 0) red[warp][3 * NP + 12 * j + i] = sum;
      }
    }
  }
}

// Block stage, executed by warp 0 only: totals of all warp partials (every lane of warp 0 gets them).
template <int NP, bool MASS>
__device__ __forceinline__ void bk_warp0_totals(Buckets<NP, MASS> &b, uint32_t (*red)[48]) {
  const int lane = threadIdx.x & 31;
  const bool act = lane < kWarps;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    b.cnt[j] = warp_sum(act ? red[lane][j] : 0u);
    const uint32_t mv = act ? red[lane][NP + j] : 0xffffffffu;
    const uint32_t m = warp_min(mv);
    b.mn[j] = m;
    b.mc[j] = warp_sum((act && mv == m) ? red[lane][2 * NP + j] : 0u);
    if (MASS) {
      uint32_t q[12];
#pragma unroll
      for (int i = 0; i < 12; ++i) q[i] = warp_sum(act ? red[lane][3 * NP + 12 * j + i] : 0u);
      b.ms[j] = fx_join(q);
    }
  }
}

// Top-k boundary search over order keys.  Restates _search_topk (pivot_search.py:93-126): NP pivots
// per pass at (j+1)/(NP+1) of [l, r], stop at a pivot with N >= k and N - n_dup < k
// (pivot_search.py:113-116).  Keys are integers, so the range always closes in <= 16 quaternary
// passes — there is no range_eps collapse and no midpoint fallback.  Invariant: cnt(l) >= k > cnt(r).
// Per pass: every warp scans its elements (only keys in (piv[0], r] can move a decision), one
// barrier, warp 0 totals the partials and decides, a second barrier broadcasts the new range.
// Exact block-wide sum of fx(v) over the elements accepted by fn(bits, idx, i, v); also counts them.
template <class Src, class Fn>
__device__ Fx block_mass(const Src &src, Fn fn, uint32_t &count, Red &R) {
  Buckets<1, true> b;
  b.cnt[0] = 0u; b.mn[0] = 0u; b.mc[0] = 0u; b.ms[0] = fx_zero();
  for_elems(src, src.n, [&](int i, uint32_t bits, uint32_t ix) {
    double v;
    if (fn(bits, ix, i, v)) { b.ms[0] = fx_add(b.ms[0], fx_from_double(v)); b.cnt[0] += 1u; }
  });
  bk_reduce(b, R);
  count = b.cnt[0];
  return b.ms[0];
}

// Bracketing pass: one pass with 255 pivots at power-of-two spacing (a 256-bucket histogram in
// shared memory, one bucket per thread for the scan).  It narrows (l, r] to the bucket that holds
// the k-th key (top-k) / the nucleus crossing (top-p) with exact counts and masses at both ends, so
// the quaternary passes that follow start from a ~256x narrower range.  Bucket b covers keys
// (l + b*2^s, l + (b+1)*2^s].  Returns true when the bucket is a single key (search finished).
__device__ __forceinline__ int bracket_shift(uint32_t w) {  // smallest s with w <= 256 * 2^s
  if (w <= (uint32_t)kBins) return 0;
  const int lg = 32 - __clz(w - 1u);  // ceil(log2(w))
  return lg - 8;
}

template <bool MASS, class Src, class Acc, class PiOf>
__device__ void bracket_pass(const Src &src, Acc acc, PiOf pi_of, uint32_t k, const Fx &T, Red &R,
                             const Fx *T_keep_all = nullptr) {
  SearchState &st = R.sm.st;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t l = st.l, r = st.r, cr = st.cr;
  const int sh = bracket_shift(r - l);
  R.hcnt[tid] = 0u;
  if (MASS) {
#pragma unroll
    for (int q = 0; q < 5; ++q) R.hms[q * kBins + tid] = 0ull;
  }
  tsync();
  for_elems(src, src.n, [&](int i, uint32_t bits, uint32_t ix) {
    const uint32_t key = key_of_bits(bits);
    if (key <= l || key > r || !acc(key, ix)) return;
    const uint32_t b = (key - l - 1u) >> sh;
    atomicAdd(&R.hcnt[b], 1u);
    if (MASS) {
      const Fx f = fx_from_double(pi_of(bits, i));
      const uint32_t pc[5] = {(uint32_t)f.w0, (uint32_t)(f.w0 >> 32), (uint32_t)f.w1,
                              (uint32_t)(f.w1 >> 32), (uint32_t)f.w2};
#pragma unroll
      for (int q = 0; q < 5; ++q)
        if (pc[q]) atomicAdd(&R.hms[q * kBins + b], (unsigned long long)pc[q]);
    }
  });
  tsync();
  // suffix scan over buckets: thread t holds bucket b = 255 - t, so a prefix over t is a suffix over b
  const int b = kBins - 1 - tid;
  const uint32_t c = R.hcnt[b];
  uint32_t ci = c;
  Fx m = fx_zero(), mi = fx_zero();
  if (MASS) {
    // normalise the 32-bit pieces (each container < 2^42) into one 192-bit value
    unsigned long long carry = 0ull;
    uint32_t pw[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const unsigned long long v = R.hms[q * kBins + b] + carry;
      pw[q] = (uint32_t)v;
      carry = v >> 32;
    }
    m = Fx{(unsigned long long)pw[0] | ((unsigned long long)pw[1] << 32),
           (unsigned long long)pw[2] | ((unsigned long long)pw[3] << 32),
           (unsigned long long)pw[4] + (carry << 32)};
    mi = m;
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t cv = __shfl_up_sync(0xffffffffu, ci, o);
    if (lane >= o) ci += cv;
    if (MASS) {
      Fx mv;
      mv.w0 = __shfl_up_sync(0xffffffffu, mi.w0, o);
      mv.w1 = __shfl_up_sync(0xffffffffu, mi.w1, o);
      mv.w2 = __shfl_up_sync(0xffffffffu, mi.w2, o);
      if (lane >= o) mi = fx_add(mi, mv);
    }
  }
  if (lane == 31) {
    R.sm.ctot[warp] = ci;
    if (MASS) R.sm.mtot[warp] = mi;
  }
  tsync();
  uint32_t above = cr;  // keys above this warp's buckets (higher buckets live in lower warps)
  Fx mab = st.Mr;
  for (int w = 0; w < warp; ++w) {
    above += R.sm.ctot[w];
    if (MASS) mab = fx_add(mab, R.sm.mtot[w]);
  }
  const uint32_t suf = above + ci;          // keys in buckets >= b, plus everything above r
  const uint32_t suf_hi = suf - c;          // keys in buckets > b
  const Fx msuf = MASS ? fx_add(mab, mi) : fx_zero();
  const Fx msuf_hi = MASS ? fx_sub(msuf, m) : fx_zero();
  if (MASS && T_keep_all && b == 0) {  // everything in range: the survivors' total
    st.Ml = msuf;
    st.cl = suf;
    st.compact = fx_ge(msuf, *T_keep_all) ? 0 : 2;  // 2 = keep all
  }
  tsync();
  if (MASS && T_keep_all && st.compact == 2) return;
  // the crossing bucket: reaches the target with itself, misses it without
  const bool in = MASS ? fx_ge(msuf, T) : (suf >= k);
  const bool hi_in = MASS ? fx_ge(msuf_hi, T) : (suf_hi >= k);
  if (in && !hi_in && c > 0u) {
    const uint32_t lo_b = l + ((uint32_t)b << sh);
    const unsigned long long hi_b = (unsigned long long)l + ((unsigned long long)(b + 1) << sh);
    st.l = lo_b;
    st.cl = suf;
    st.r = hi_b < (unsigned long long)r ? (uint32_t)hi_b : r;
    st.cr = suf_hi;
    if (MASS) { st.Ml = msuf; st.Mr = msuf_hi; }
    if (sh == 0) {  // single-key bucket: done
      st.done = 1u; st.K = lo_b + 1u; st.n_gt = suf_hi; st.n_eq = c;
      if (MASS) st.H = msuf_hi;
    }
    st.iters += 1;
  }
  tsync();
}

template <int NP, class Src>
__device__ KRes search_k(const Src &src, uint32_t l, uint32_t r, uint32_t cl, uint32_t cr, uint32_t k,
                         Red &R) {
  SearchState &st = R.sm.st;
  if (threadIdx.x == 0) {
    st.l = l; st.r = r; st.cl = cl; st.cr = cr; st.done = 0u; st.iters = 0; st.compact = 0; st.n_act = 0u;
  }
  tsync();
  const Fx zero = fx_zero();
  if (r - l > (uint32_t)(4 * kBins)) {
    bracket_pass<false>(src, [&](uint32_t, uint32_t) { return true; },
                        [&](uint32_t, int) { return 0.0; }, k, zero, R);
    if (threadIdx.x == 0 && !st.done) {
      const uint32_t n_in = st.cl - st.cr;
      if ((int)n_in <= R.act_cap_k && 2 * (int)n_in <= src.n) st.compact = 1;
    }
    tsync();
  }
  bool act = false;  // searching the compacted active set instead of src
  for (;;) {
    l = st.l; r = st.r; cr = st.cr;
    if (st.done || r - l <= 1u) break;
    if (st.compact && !act) {
      // keep only the keys that can still matter: (l, r]  (order is irrelevant to counts)
      for_elems_warp(src, src.n, [&](int, bool valid, uint32_t bits, uint32_t) {
        const uint32_t key = key_of_bits(bits);
        const bool keep = valid && key > l && key <= r;
        const uint32_t pos = warp_reserve(&st.n_act, keep);
        if (keep) R.act_key[pos] = key;
      });
      act = true;
      tsync();
    }
    const int n = act ? (int)st.n_act : src.n;
    uint32_t piv[NP];
    make_pivots<NP>(l, r, piv);
    Buckets<NP, false> b;
    bk_init(b);
    // only keys inside (piv[0], r] can move a decision; everything above r is the known cr
    if (act) {
      for (int i = threadIdx.x; i < n; i += kThreads) {
        const uint32_t key = R.act_key[i];
        if (key > piv[0] && key <= r) bk_add(b, piv, key, zero);
      }
    } else {
      for_elems(src, n, [&](int, uint32_t bits, uint32_t) {
        const uint32_t key = key_of_bits(bits);
        if (key > piv[0] && key <= r) bk_add(b, piv, key, zero);
      });
    }
    uint32_t(*red)[48] = R.sm.red[R.par];
    R.par ^= 1;
    bk_warp_partials(b, red);
    tsync();
    if (threadIdx.x < 32) {
      bk_warp0_totals(b, red);
      uint32_t cnt[NP], mn[NP], mc[NP];
      uint32_t c = cr, m = 0xffffffffu, x = 0u;
#pragma unroll
      for (int j = NP - 1; j >= 0; --j) {
        c += b.cnt[j];
        if (b.cnt[j] > 0u) { m = b.mn[j]; x = b.mc[j]; }
        cnt[j] = c; mn[j] = m; mc[j] = x;
      }
      int J = -1;  // largest pivot still holding >= k keys above it
#pragma unroll
      for (int j = 0; j < NP; ++j) J = (cnt[j] >= k) ? j : J;
      // pick the J and J+1 entries with unrolled selects (no dynamically indexed local arrays)
      uint32_t cJ = 0u, mJ = 0u, xJ = 0u, pJ = 0u, cJ1 = 0u, pJ1 = 0u;
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        if (j == J) { cJ = cnt[j]; mJ = mn[j]; xJ = mc[j]; pJ = piv[j]; }
        if (j == J + 1) { cJ1 = cnt[j]; pJ1 = piv[j]; }
      }
      if (threadIdx.x == 0) {
        st.iters += 1;
        if (J >= 0 && cJ - xJ < k) {
          st.done = 1u; st.K = mJ; st.n_gt = cJ - xJ; st.n_eq = xJ;
        } else {
          if (J >= 0) { st.l = pJ; st.cl = cJ; }
          if (J + 1 < NP) { st.r = pJ1; st.cr = cJ1; }
          const uint32_t n_in = st.cl - st.cr;
          if (!act && (int)n_in <= R.act_cap_k && 2 * (int)n_in <= n) st.compact = 1;
        }
      }
    }
    tsync();
  }
  const KRes res = st.done ? KRes{st.K, st.n_gt, st.n_eq, st.iters}
                           : KRes{st.r, st.cr, st.cl - st.cr, st.iters};
  tsync();
  return res;
}

struct PRes {
  uint32_t K;      // boundary key of the nucleus
  uint32_t n_gt;   // survivors strictly above K
  uint32_t n_eq;   // survivors equal to K
  Fx H;            // exact mass strictly above K
  int iters;
  bool keep_all;   // p >= fsum(all survivors): no truncation (oracle.py:45-46)
  Fx total;        // exact mass of all survivors
};

// Top-p boundary search.  Restates _search_topp + _resolve_topp (pivot_search.py:159-232) with logit
// keys as pivots and exact masses: the crossing cluster (fsum(head) < p <= fsum(head + cluster),
// pivot_search.py:177-191) is found directly, no resolve walk.  Invariant: M(l) >= T > M(r).
// The survivors' total mass is computed here (by the bracketing pass when the range is wide, else by
// one reduction); when p >= fsum(total) the result is keep_all.
template <int NP, class Src, class InS, class PiOf, class PiKey>
__device__ PRes search_p(const Src &src, uint32_t l, uint32_t r, const Fx &T, const Fx &Tsp, InS in_s,
                         PiOf pi_of, PiKey pi_key, Red &R) {
  SearchState &st = R.sm.st;
  uint32_t cl = 0u, cr = 0u;
  Fx Ml = fx_zero(), Mr = fx_zero();
  if (threadIdx.x == 0) {
    st.l = l; st.r = r; st.cl = 0u; st.cr = 0u; st.Ml = Ml; st.Mr = Mr; st.done = 0u; st.iters = 0;
    st.compact = 0; st.n_act = 0u;
  }
  tsync();
  if (r - l > (uint32_t)(4 * kBins)) {
    bracket_pass<true>(src, in_s, pi_of, 0u, T, R, &Tsp);
    if (st.compact == 2) {  // keep everything
      PRes res{};
      res.keep_all = true;
      res.total = st.Ml;
      tsync();
      return res;
    }
    if (threadIdx.x == 0 && !st.done) {
      const uint32_t n_in = st.cl - st.cr;
      if ((int)n_in <= R.act_cap_p && 2 * (int)n_in <= src.n) st.compact = 1;
    }
    tsync();
  } else {
    uint32_t cnt;
    const Fx tot = block_mass(src, [&](uint32_t bits, uint32_t ix, int i, double &v) {
      if (!in_s(key_of_bits(bits), ix)) return false;
      v = pi_of(bits, i); return true; }, cnt, R);
    if (!fx_ge(tot, Tsp)) {
      PRes res{};
      res.keep_all = true;
      res.total = tot;
      return res;
    }
    if (threadIdx.x == 0) { st.cl = cnt; st.Ml = tot; }
    tsync();
  }
  bool act = false;
  for (;;) {
    l = st.l; r = st.r; cr = st.cr;
    if (st.done || r - l <= 1u) break;
    Mr = st.Mr;
    if (st.compact && !act) {
      // survivors in (l, r] with their probabilities: later passes need neither src nor exp()
      for_elems_warp(src, src.n, [&](int i, bool valid, uint32_t bits, uint32_t ix) {
        const uint32_t key = key_of_bits(bits);
        const bool keep = valid && key > l && key <= r && in_s(key, ix);
        const uint32_t pos = warp_reserve(&st.n_act, keep);
        if (keep) { R.act_key[pos] = key; R.act_pi[pos] = pi_of(bits, i); }
      });
      act = true;
      tsync();
    }
    const int n = act ? (int)st.n_act : src.n;
    uint32_t piv[NP];
    make_pivots<NP>(l, r, piv);
    Buckets<NP, true> b;
    bk_init(b);
    if (act) {
      for (int i = threadIdx.x; i < n; i += kThreads) {
        const uint32_t key = R.act_key[i];
        if (key > piv[0] && key <= r) bk_add(b, piv, key, fx_from_double(R.act_pi[i]));
      }
    } else {
      for_elems(src, n, [&](int i, uint32_t bits, uint32_t ix) {
        const uint32_t key = key_of_bits(bits);
        if (key > piv[0] && key <= r && in_s(key, ix)) bk_add(b, piv, key, fx_from_double(pi_of(bits, i)));
      });
    }
    uint32_t(*red)[48] = R.sm.red[R.par];
    R.par ^= 1;
    bk_warp_partials(b, red);
    tsync();
    if (threadIdx.x < 32) {
      bk_warp0_totals(b, red);
      uint32_t cnt[NP], mn[NP], mc[NP];
      Fx M[NP];
      uint32_t c = cr, m = 0xffffffffu, x = 0u;
      Fx sacc = Mr;
#pragma unroll
      for (int j = NP - 1; j >= 0; --j) {
        c += b.cnt[j];
        if (b.cnt[j] > 0u) { m = b.mn[j]; x = b.mc[j]; }
        sacc = fx_add(sacc, b.ms[j]);
        cnt[j] = c; mn[j] = m; mc[j] = x; M[j] = sacc;
      }
      int J = -1;  // largest pivot whose mass above still reaches p
#pragma unroll
      for (int j = 0; j < NP; ++j) J = fx_ge(M[j], T) ? j : J;
      bool done = false;
      Fx HJ = fx_zero();
      uint32_t KJ = 0u, gJ = 0u, eJ = 0u, lJ = 0u, clJ = 0u, rJ = 0u, crJ = 0u;
      Fx MlJ = fx_zero(), MrJ = fx_zero();
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        if (j == J) {
          HJ = fx_sub(M[j], fx_mul_u32(fx_from_double(pi_key(mn[j])), mc[j]));
          done = !fx_ge(HJ, T);
          KJ = mn[j]; gJ = cnt[j] - mc[j]; eJ = mc[j];
          lJ = piv[j]; clJ = cnt[j]; MlJ = M[j];
        }
        if (j == J + 1) { rJ = piv[j]; crJ = cnt[j]; MrJ = M[j]; }
      }
      if (threadIdx.x == 0) {
        st.iters += 1;
        if (done) {
          st.done = 1u; st.K = KJ; st.n_gt = gJ; st.n_eq = eJ; st.H = HJ;
        } else {
          if (J >= 0) { st.l = lJ; st.cl = clJ; st.Ml = MlJ; }
          if (J + 1 < NP) { st.r = rJ; st.cr = crJ; st.Mr = MrJ; }
          const uint32_t n_in = st.cl - st.cr;
          if (!act && (int)n_in <= R.act_cap_p && 2 * (int)n_in <= n) st.compact = 1;
        }
      }
    }
    tsync();
  }
  const PRes res = st.done ? PRes{st.K, st.n_gt, st.n_eq, st.H, st.iters, false, fx_zero()}
                           : PRes{st.r, st.cr, st.cl - st.cr, st.Mr, st.iters, false, fx_zero()};
  tsync();
  return res;
}

__device__ __forceinline__ int nth_set_bit(uint32_t m, uint32_t n) {  // n >= 1
  for (uint32_t t = 1u; t < n; ++t) m &= m - 1u;
  return __ffs((int)m) - 1;
}

// Index of the c-th (1-based) element with key K in index order, over an index-ordered source.
// Warp-contiguous segments: ballot/popc counts per warp, a 16-entry prefix, one warp re-scans.
// This is the duplicate-trimming rule of _apply_plan (pipeline.py:53-56): occurrences beyond n_keep,
// counted left to right, are dropped.
template <class Src>
__device__ uint32_t select_nth_eq(const Src &src, uint32_t K, uint32_t c, Red &R) {
  TailSmem &sm = R.sm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = src.n;
  const int seg = ((n + kWarps - 1) / kWarps + 31) & ~31;
  const int beg = warp * seg, end = min(n, beg + seg);
  uint32_t cnt = 0u;
  for (int base = beg; base < end; base += 32 * kLd) {  // kLd rows of 32 loads in flight per warp
    uint32_t b[kLd];
#pragma unroll
    for (int j = 0; j < kLd; ++j) {
      const int i = base + 32 * j + lane;
      uint32_t ix;
      b[j] = 0u;
      if (i < end) src.get(i, b[j], ix);
    }
#pragma unroll
    for (int j = 0; j < kLd; ++j) {
      const int i = base + 32 * j + lane;
      cnt += __popc(__ballot_sync(0xffffffffu, i < end && key_of_bits(b[j]) == K));
    }
  }
  if (lane == 0) sm.sel[warp] = cnt;
  tsync();
  if (threadIdx.x == 0) {
    uint32_t acc = 0u;
    int w = 0;
    for (; w < kWarps; ++w) {
      if (acc + sm.sel[w] >= c) break;
      acc += sm.sel[w];
    }
    sm.u[0] = (uint32_t)w;
    sm.u[1] = c - acc;
    sm.u[2] = kNoCut;
  }
  tsync();
  const int w_star = (int)sm.u[0];
  if (warp == w_star) {
    uint32_t need = sm.u[1];
    bool found = false;
    for (int base = beg; base < end && !found; base += 32 * kLd) {
      uint32_t b[kLd], x[kLd];
#pragma unroll
      for (int j = 0; j < kLd; ++j) {
        const int i = base + 32 * j + lane;
        b[j] = x[j] = 0u;
        if (i < end) src.get(i, b[j], x[j]);
      }
#pragma unroll
      for (int j = 0; j < kLd; ++j) {
        const int i = base + 32 * j + lane;
        const uint32_t bal = __ballot_sync(0xffffffffu, i < end && key_of_bits(b[j]) == K);
        const uint32_t pc = (uint32_t)__popc(bal);
        if (!found) {
          if (pc >= need) {
            if (lane == nth_set_bit(bal, need)) sm.u[2] = x[j];
            found = true;
          } else {
            need -= pc;
          }
        }
      }
    }
  }
  tsync();
  const uint32_t res = sm.u[2];
  tsync();
  return res;
}

// Visits every element of a row in global memory, fn(i, valid, bits) with fp32-expanded bits, called by
// all lanes (warp-converged, for match_any aggregation).  16-byte vector loads, kLd in flight per
// thread, when the row is aligned.
template <typename T, class Fn>
__device__ __forceinline__ void for_row_warp(const T *in, int V, Fn fn) {
  using VT = typename Vec<T>::type;
  constexpr int W = Vec<T>::W;
  const int tid = threadIdx.x;
  if (((uintptr_t)in % 16) == 0 && V % W == 0) {
    const VT *p = reinterpret_cast<const VT *>(in);
    const int nv = V / W;
    for (int b0 = 0; b0 < nv; b0 += kThreads * kLd) {
      VT r[kLd];
#pragma unroll
      for (int j = 0; j < kLd; ++j) {
        const int vi = b0 + j * kThreads + tid;
        if (vi < nv) r[j] = __ldcg(p + vi);
      }
#pragma unroll
      for (int j = 0; j < kLd; ++j) {
        const int vi = b0 + j * kThreads + tid;
#pragma unroll
        for (int w = 0; w < W; ++w) fn(vi * W + w, vi < nv, vi < nv ? lane_bits<T>(r[j], w) : 0u);
      }
    }
  } else {
    for (int b0 = 0; b0 < V; b0 += kThreads * kLd) {
      uint32_t r[kLd];
#pragma unroll
      for (int j = 0; j < kLd; ++j) {
        const int i = b0 + j * kThreads + tid;
        r[j] = i < V ? Elem<T>::bits(in[i]) : 0u;
      }
#pragma unroll
      for (int j = 0; j < kLd; ++j) fn(b0 + j * kThreads + tid, b0 + j * kThreads + tid < V, r[j]);
    }
  }
}

struct DistinctRes {
  bool ok;        // false: too many distinct values, use the pivot search
  bool keep_all;  // p >= fsum(all)
  uint32_t K, n_gt, n_eq, j;  // boundary key, entries above it, copies of it, copies kept
  double mx;      // outlier mass (sigma_trunc.py:121), for the hit metric
  bool hit;       // outlier mass > p
};

// Top-p over a whole row through its distinct values (pipeline.py:161-196 semantics of oracle.py:37-67).
// Equal logits have equal probabilities, so the nucleus only needs each distinct value's count: one
// pass counts them into a shared-memory hash table (warp-aggregated with match_any), then the
// distinct values are sorted descending (bin counting sort) and fp64 exp, the exact normaliser
// D = sum count * exp(v - m), probabilities fl(e / D) and the exact prefix masses are computed per
// distinct value.  Rows with few distinct values (bf16 / quantised logits) cost one row pass instead
// of a pivot search with an fp64 exp per element per pass.  tk/tc: table of cap (power of two)
// entries; lk/lc, sk/sc: kCapC-entry lists; hc/he: kNB bins; ev: kCapC doubles.
template <typename T>
__device__ __noinline__ DistinctRes distinct_topp(const Params &P, int row, const T *in, int V, double m, const RowPlan &pl, uint32_t *tk,
                                     uint32_t *tc, uint32_t cap, uint32_t *lk, uint32_t *lc, uint32_t *sk,
                                     uint32_t *sc, uint32_t *hc, uint32_t *he, double *ev, TailSmem &sm) {
  // lk/lc: compacted table, then the sorted result; sk/sc: grouped by bin
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t lg = 31u - (uint32_t)__clz((int)cap);
  const uint32_t limit = min(cap / 2u, (uint32_t)kCapC);
  DistinctRes res{};
  for (uint32_t h = tid; h < cap; h += kThreads) { tk[h] = 0u; tc[h] = 0u; }
  for (int i = tid; i < kNB; i += kThreads) hc[i] = 0u;
  if (tid == 0) { sm.nd = 0u; sm.dabort = 0u; sm.u[4] = 0u; sm.dkmin = 0xffffffffu; sm.dkmax = 0u; }
  tsync();
  // 1. count every distinct key (keys of finite logits are >= 1; 0 marks an empty slot).  Elements go
  //    in batches: the table probes of a batch are independent loads, and keys already present (all
  //    but the first copy of each value) take one atomic add; new keys go through the CAS insert.
  auto insert_slow = [&](uint32_t key) {
    uint32_t h = (key * 0x9E3779B1u) >> (32u - lg);
    for (uint32_t probe = 0; probe < cap; ++probe) {
      const uint32_t cur = *(volatile uint32_t *)&tk[h];
      if (cur == key) { atomicAdd(&tc[h], 1u); return; }
      if (cur != 0u) { h = (h + 1u) & (cap - 1u); continue; }
      if (sm.dabort) return;
      const uint32_t old = atomicCAS(&tk[h], 0u, key);
      if (old == 0u || old == key) {
        atomicAdd(&tc[h], 1u);
        if (old == 0u && atomicAdd(&sm.nd, 1u) >= limit) sm.dabort = 1u;
        return;
      }
      h = (h + 1u) & (cap - 1u);
    }
  };
  {
    using VT = typename Vec<T>::type;
    constexpr int W = Vec<T>::W;
    if (((uintptr_t)in % 16) == 0 && V % W == 0) {
      const VT *pv = reinterpret_cast<const VT *>(in);
      const int nv = V / W;
      for (int v0 = tid; v0 < nv; v0 += kThreads * 2) {
        VT r[2];
#pragma unroll
        for (int j = 0; j < 2; ++j)
          if (v0 + j * kThreads < nv) r[j] = __ldcg(pv + v0 + j * kThreads);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if (v0 + j * kThreads >= nv) continue;
          uint32_t key[W], h[W], cur[W];
#pragma unroll
          for (int w = 0; w < W; ++w) {
            key[w] = key_of_bits(lane_bits<T>(r[j], w));
            h[w] = (key[w] * 0x9E3779B1u) >> (32u - lg);
          }
#pragma unroll
          for (int w = 0; w < W; ++w) cur[w] = *(volatile uint32_t *)&tk[h[w]];
#pragma unroll
          for (int w = 0; w < W; ++w) {
            if (cur[w] == key[w]) atomicAdd(&tc[h[w]], 1u);
            else insert_slow(key[w]);
          }
        }
      }
    } else {
      for (int i = tid; i < V; i += kThreads) insert_slow(key_of_bits(Elem<T>::bits(in[i])));
    }
  }
  tsync();
  QRITA_TSTAMP(10);
  if (sm.dabort) return res;  // block-uniform
  const uint32_t nd = sm.nd;
  // 2. compact the table; key range of the distinct values
  uint32_t kmin = 0xffffffffu, kmax = 0u;
  for (uint32_t h0 = 0; h0 < cap; h0 += kThreads) {
    const uint32_t h = h0 + tid;
    const uint32_t key = h < cap ? tk[h] : 0u;
    const bool keep = key != 0u;
    const uint32_t pos = warp_reserve(&sm.u[4], keep);
    if (keep) { lk[pos] = key; lc[pos] = tc[h]; kmin = min(kmin, key); kmax = max(kmax, key); }
  }
  kmin = warp_min(kmin);
  kmax = warp_max(kmax);
  if (lane == 0) { atomicMin(&sm.dkmin, kmin); atomicMax(&sm.dkmax, kmax); }
  tsync();
  kmin = sm.dkmin;
  kmax = sm.dkmax;
  // 3. sort descending: counting sort over key bins, then rank inside each bin (keys are distinct)
  const int sh = bin_shift(kmax - kmin + 1u);
  auto bin_of = [&](uint32_t key) -> uint32_t { return (key - kmin) >> sh; };
  for (uint32_t i = tid; i < nd; i += kThreads) atomicAdd(&hc[bin_of(lk[i])], 1u);
  tsync();
  {
    uint32_t c4[4], loc = 0u;
#pragma unroll
    for (int j = 0; j < 4; ++j) { c4[j] = hc[kNB - 1 - 4 * tid - j]; loc += c4[j]; }
    uint32_t tot;
    uint32_t run = block_exscan_u32(loc, sm.scan_u, tot);
#pragma unroll
    for (int j = 0; j < 4; ++j) { he[kNB - 1 - 4 * tid - j] = run; run += c4[j]; }
  }
  tsync();
  for (uint32_t i = tid; i < nd; i += kThreads) {  // group by bin (order inside a bin arbitrary)
    const uint32_t key = lk[i];
    const uint32_t pos = atomicAdd(&he[bin_of(key)], 1u);
    sk[pos] = key;
    sc[pos] = lc[i];
  }
  tsync();
  for (uint32_t q = tid; q < nd; q += kThreads) {  // rank inside the bin: he[b] is now the bin's end
    const uint32_t key = sk[q], b = bin_of(key);
    const uint32_t e = he[b], c = hc[b];
    uint32_t r = 0u;
    for (uint32_t j = e - c; j < e; ++j) r += sk[j] > key ? 1u : 0u;
    lk[e - c + r] = key;
    lc[e - c + r] = sc[q];
  }
  tsync();
  // sorted: (lk, lc)[0, nd) by key descending
  sk = lk;
  sc = lc;
  QRITA_TSTAMP(11);
  // 4. exact normaliser and prefix masses over the sorted distinct values (thread t owns a
  //    contiguous run of E entries)
  const int E = ((int)nd + kThreads - 1) / kThreads;
  const int q0 = tid * E;
  Fx dl = fx_zero();
  uint32_t cl = 0u;
  for (int j = 0; j < E; ++j) {
    const int q = q0 + j;
    if (q < (int)nd) {
      const double e = exp(value_of_key(sk[q]) - m);
      ev[q] = e;
      dl = fx_add(dl, fx_mul_u32(fx_from_double(e), sc[q]));
      cl += sc[q];
    }
  }
  Fx Dx;
  (void)block_exscan_fx(dl, sm.scan_f[0], Dx);
  const double D = fx_to_double(Dx);
  Fx ml = fx_zero();
  for (int j = 0; j < E; ++j) {
    const int q = q0 + j;
    if (q < (int)nd) {
      const double pi = ev[q] / D;
      ev[q] = pi;
      ml = fx_add(ml, fx_mul_u32(fx_from_double(pi), sc[q]));
    }
  }
  Fx Mtot;
  uint32_t ctot;
  Fx pre = block_exscan_fx(ml, sm.scan_f[1], Mtot);
  uint32_t cpre = block_exscan_u32(cl, sm.scan_u2, ctot);
  if (tid == 0) { sm.L = 0xffffffffu; sm.dMx = fx_zero(); }
  tsync();
  for (int j = 0; j < E; ++j) {
    const int q = q0 + j;
    if (q < (int)nd) {
      const Fx mass = fx_mul_u32(fx_from_double(ev[q]), sc[q]);
      const Fx incl = fx_add(pre, mass);
      // outliers (key >= threshold) are a prefix of the sorted values: the last one holds their mass
      if (pl.has_thr && sk[q] >= pl.key_thr && (q + 1 == (int)nd || sk[q + 1] < pl.key_thr)) sm.dMx = incl;
      if (fx_ge(incl, pl.t_p) && !fx_ge(pre, pl.t_p)) {  // the (unique) crossing value
        sm.L = (uint32_t)q; sm.dK = sk[q]; sm.dngt = cpre; sm.dneq = sc[q]; sm.dH = pre;
      }
      pre = incl;
      cpre += sc[q];
    }
  }
  tsync();
  QRITA_TSTAMP(12);
  res.ok = true;
  res.mx = fx_to_double(sm.dMx);
  res.hit = fx_ge(sm.dMx, pl.t_sp);
  res.keep_all = !fx_ge(Mtot, pl.t_sp) || sm.L == 0xffffffffu;
  if (!res.keep_all) {
    res.K = sm.dK; res.n_gt = sm.dngt; res.n_eq = sm.dneq;
    // smallest j with fsum(head + j * p_b) >= p (_min_dup_count, pivot_search.py:143-156), exactly
    const double pb = ev[sm.L];
    const Fx fb = fx_from_double(pb);
    const Fx H = sm.dH;
    const double jd = ceil(fx_to_double(fx_sub(pl.t_p, H)) / pb);
    uint32_t j = (jd < 1.0) ? 1u : (jd > (double)res.n_eq ? res.n_eq : (uint32_t)jd);
    while (j > 1u && fx_ge(fx_add(H, fx_mul_u32(fb, j - 1u)), pl.t_p)) --j;
    while (j < res.n_eq && !fx_ge(fx_add(H, fx_mul_u32(fb, j)), pl.t_p)) ++j;
    res.j = j;
  }
  tsync();
  return res;
}

// select_nth_eq over a row in global memory with 16-byte vector loads (aligned rows).  Pass 1 counts
// the matches of every 32-vector block (kLdRow blocks in flight per warp) into blk[] (nblk <= cap
// words of shared memory); warp 0 scans the block counts; one warp reloads the single block that
// holds the c-th copy.  Returns kNoCut if the row has more blocks than blk holds (caller falls back).
constexpr int kLdRow = 8;
template <typename T>
__device__ uint32_t select_nth_eq_row(const T *in, int V, uint32_t K, uint32_t c, TailSmem &sm, uint32_t *blk,
                                      int blk_cap, bool &ok) {
  using VT = typename Vec<T>::type;
  constexpr int W = Vec<T>::W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const VT *pv = reinterpret_cast<const VT *>(in);
  const int nv = V / W;
  const int nblk = (nv + 31) / 32;
  ok = nblk <= blk_cap;
  if (!ok) return kNoCut;  // uniform
  const VecCmp<T> cmp(K);
  auto mask_of = [&](VT r) -> uint32_t {
    uint32_t gt, eq;
    cmp.masks(r, gt, eq);
    return eq;
  };
  // pass 1: block b = 32 consecutive vectors; warp w takes blocks w, w + 8, ... (kLdRow at a time)
  for (int b0 = warp; b0 < nblk; b0 += kWarps * kLdRow) {
    uint32_t cnt[kLdRow];
#pragma unroll
    for (int j = 0; j < kLdRow; ++j) {
      const int vi = (b0 + j * kWarps) * 32 + lane;
      cnt[j] = vi < nv ? (uint32_t)__popc(mask_of(__ldcg(pv + vi))) : 0u;
    }
#pragma unroll
    for (int j = 0; j < kLdRow; ++j) {
      const uint32_t t = warp_sum(cnt[j]);
      if (lane == 0 && b0 + j * kWarps < nblk) blk[b0 + j * kWarps] = t;
    }
  }
  tsync();
  // warp 0: first block whose inclusive prefix reaches c
  if (warp == 0) {
    const int per = (nblk + 31) / 32;
    uint32_t loc = 0u;
    for (int i = 0; i < per; ++i) {
      const int b = lane * per + i;
      if (b < nblk) loc += blk[b];
    }
    uint32_t incl = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    uint32_t before = incl - loc;
    const bool mine = before < c && incl >= c;
    const uint32_t who = __ballot_sync(0xffffffffu, mine);
    if (mine) {
      for (int i = 0; i < per; ++i) {
        const int b = lane * per + i;
        const uint32_t t = b < nblk ? blk[b] : 0u;
        if (before + t >= c) { sm.u[0] = (uint32_t)b; sm.u[1] = c - before; break; }
        before += t;
      }
    }
    if (who == 0u && lane == 0) { sm.u[0] = 0xffffffffu; sm.u[1] = 0u; }
  }
  tsync();
  if (warp == 0) {
    const uint32_t b = sm.u[0];
    uint32_t res = kNoCut;
    if (b != 0xffffffffu) {
      const uint32_t need = sm.u[1];
      const int vi = (int)b * 32 + lane;
      const uint32_t mk = vi < nv ? mask_of(__ldcg(pv + vi)) : 0u;
      const uint32_t pc = (uint32_t)__popc(mk);
      uint32_t incl = pc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (incl >= need && incl - pc < need) res = (uint32_t)(vi * W + nth_set_bit(mk, need - (incl - pc)));
      res = warp_min(res);
    }
    if (lane == 0) sm.u[2] = res;
  }
  tsync();
  const uint32_t res = sm.u[2];
  tsync();
  return res;
}

__device__ __forceinline__ bool kept_by(uint32_t key, uint32_t idx, uint32_t K, uint32_t cut) {
  return key > K || (key == K && idx <= cut);
}

// Full-row output pass.  how: 0 = kept values only (background already -inf), 1 = every element,
// 2 = -inf where not kept (in-place).
template <typename T>
__device__ void write_row(const T *in, T *out, int V, uint32_t K, uint32_t cut, int how) {
  using VT = typename Vec<T>::type;
  constexpr int W = Vec<T>::W;
  if (((uintptr_t)in % 16) == 0 && ((uintptr_t)out % 16) == 0 && V % W == 0) {
    const VT *pi = reinterpret_cast<const VT *>(in);
    VT *po = reinterpret_cast<VT *>(out);
    const int nv = V / W;
    const VecCmp<T> cmp(K);
    for (int v0 = threadIdx.x; v0 < nv; v0 += kThreads * kLd) {
      VT r[kLd];
#pragma unroll
      for (int j = 0; j < kLd; ++j)
        if (v0 + j * kThreads < nv) r[j] = __ldcg(pi + v0 + j * kThreads);
#pragma unroll
      for (int j = 0; j < kLd; ++j) {
        const int vi = v0 + j * kThreads;
        if (vi >= nv) continue;
        uint32_t gt, eq;
        cmp.masks(r[j], gt, eq);
        uint32_t kp = gt;
        if (eq) {  // the boundary value: copies up to index `cut` are kept
#pragma unroll
          for (int w = 0; w < W; ++w)
            if (((eq >> w) & 1u) && (uint32_t)(vi * W + w) <= cut) kp |= 1u << w;
        }
        constexpr uint32_t kAll = (1u << W) - 1u;
        const T *ie = reinterpret_cast<const T *>(&r[j]);
        if (how == 0) {
          if (kp) {
#pragma unroll
            for (int w = 0; w < W; ++w)
              if ((kp >> w) & 1u) out[vi * W + w] = ie[w];
          }
        } else if (kp == kAll) {
          if (how == 1) po[vi] = r[j];
        } else if (kp == 0u) {
          po[vi] = neg_inf_vec<T>();
        } else {
          VT o = r[j];
          T *oe = reinterpret_cast<T *>(&o);
#pragma unroll
          for (int w = 0; w < W; ++w)
            if (!((kp >> w) & 1u)) oe[w] = Elem<T>::neg_inf();
          po[vi] = o;
        }
      }
    }
    return;
  }
  for (int i0 = threadIdx.x; i0 < V; i0 += kThreads * kLd) {
    T v[kLd];
#pragma unroll
    for (int j = 0; j < kLd; ++j) {
      const int i = i0 + j * kThreads;
      if (i < V) v[j] = in[i];
    }
#pragma unroll
    for (int j = 0; j < kLd; ++j) {
      const int i = i0 + j * kThreads;
      if (i >= V) continue;
      const bool kp = kept_by(key_of_bits(Elem<T>::bits(v[j])), (uint32_t)i, K, cut);
      if (how == 0) { if (kp) out[i] = v[j]; }
      else if (how == 1) { out[i] = kp ? v[j] : Elem<T>::neg_inf(); }
      else { if (!kp) out[i] = Elem<T>::neg_inf(); }
    }
  }
}


// Row tail proper, run by the tail thread group (kThreads threads, tsync barriers) once the row's
// outliers X = (xb, xi)[0, n_c) are in shared memory (in any order; only when they fit: n_c <= kCapX
// and !overflow) and its aggregates are known: search + duplicate trimming + output of
// pipeline.py:88-239 with the oracle's semantics (oracle.py:70-89).  `work` is kWorkBytes of shared
// memory.  Writes the kept logits (the -inf / copy background was written by the streaming pass,
// except for top-p-only and in-place rows, which are written here in full), kept_count, metrics and
// the non-finite status.
template <typename T, int NP>
__device__ void tail_resolve(const Params &P, int row, const RowPlan &pl, uint32_t *xb, uint32_t *xi,
                             uint8_t *work, TailSmem &sm, uint32_t n_c, bool overflow, uint32_t maxkey,
                             uint32_t minkey, uint32_t nf_col, uint32_t xcap, const uint32_t *gxb = nullptr,
                             const uint32_t *gxi = nullptr, uint32_t gcap = 0u,
                             const uint32_t *hist_in = nullptr, int bsh_in = 0,
                             size_t work_bytes = (size_t)kWorkBytes) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int V = P.V;
  const T *in = (const T *)P.logits + (size_t)row * P.ld_in;
  T *out = (T *)P.out + (size_t)row * P.ld_out;
  const bool inplace = (P.flags & QRITA_INPLACE) != 0;
  const bool nodup = (P.flags & QRITA_NO_DUP) != 0;
  const bool force_fb = (P.flags & QRITA_FORCE_FALLBACK) != 0;
  uint32_t *sb = (uint32_t *)work;       // [kCapS] survivor bits
  uint32_t *si = sb + kCapS;             // [kCapS] survivor indices
  double *sp = (double *)(si + kCapS);   // [kCapS] survivor exp / probability
  double *ap = sp + kCapS;               // [kCapA] active-set probabilities (top-p search)
  uint32_t *ak = (uint32_t *)(ap + kCapA);  // [kCapA] active-set keys (3*kCapA keys for top-k)
  // bin-sort layout of the same work area
  uint32_t *hc = (uint32_t *)work;       // [kNB] outliers per key bin
  uint32_t *he = hc + kNB;               // [kNB] bin starts (descending order) -> cursors -> ends
  uint32_t *cb = he + kNB;               // [kCapC] candidates grouped by bin: bits
  uint32_t *ci = cb + kCapC;             //                                     indices
  uint32_t *db = ci + kCapC;             // [kCapC] candidates sorted (key desc, index asc): bits
  uint32_t *di = db + kCapC;             //                                                  indices
  double *ev = (double *)cb;             // [kCapC] survivor exp values (after the sort)
  const uint32_t lo_row = minkey ? minkey - 1u : 0u;  // below every key of the row

  qrita_row_metrics met;
  memset(&met, 0, sizeof(met));
  if (nf_col != 0xffffffffu) {  // validate_batch (core.py:124-128): reported, row left undefined
    uint32_t first = 0xffffffffu;  // exact first non-finite column (error path only)
    for (int i = (int)nf_col + tid; i < V; i += kThreads)
      if (bits_nonfinite(Elem<T>::bits(in[i]))) { first = (uint32_t)i; break; }
    first = warp_min(first);
    if (lane == 0) sm.sel[warp] = first;
    tsync();
    if (tid == 0) {
      for (int w = 0; w < kWarps; ++w) first = min(first, sm.sel[w]);
      P.status[row] |= ST_NONFINITE;
      P.nf_col[row] = (int32_t)first;
    }
    return;
  }
  const int mode = pl.mode;
  if (mode == MODE_INVALID) return;
  if (mode == MODE_PASS) {  // _passthrough, pipeline.py:81-85 (the stream already copied the row)
    if (tid == 0) {
      met.kept_count = V;
      if (P.kept_count) P.kept_count[row] = V;
      if (P.metrics) P.metrics[row] = met;
    }
    return;
  }

  const bool sigma = pl.has_thr != 0;
  const double m = value_of_key(maxkey);
  met.outlier_count = sigma ? (int32_t)n_c : 0;
  // X = (xb, xi)[0, xcap) in shared memory, continued by (gxb, gxi)[0, gcap) in HBM (fused kernel)
  const bool x_fits = sigma && !overflow && n_c <= xcap;
  const bool x_fits_all = sigma && !overflow && n_c <= xcap + gcap;
  auto x_bits = [&](uint32_t i) -> uint32_t { return i < xcap ? xb[i] : __ldcg(gxb + (i - xcap)); };
  auto x_idx = [&](uint32_t i) -> uint32_t { return i < xcap ? xi[i] : __ldcg(gxi + (i - xcap)); };
  // bin-sort resolve: sigma hit (count > k, sigma_trunc.py:127-133) of a top-k / top-k+top-p row
  const bool bins = x_fits_all && NP == 3 && !force_fb && !nodup && (mode == MODE_TOPK || mode == MODE_TOPKP) &&
                    pl.k <= (int64_t)kCapC && n_c > (uint32_t)pl.k;
  const uint32_t bl = pl.key_thr ? pl.key_thr - 1u : 0u;  // every outlier key is > bl
  // key bins (bl + b*2^bsh, bl + (b+1)*2^bsh], the last one open above: monotone in the key
  const int bsh = hist_in ? bsh_in : bin_shift(maxkey - bl);
  auto bin_of = [&](uint32_t key) -> uint32_t {
    const uint32_t b = (key - bl - 1u) >> bsh;
    return b < (uint32_t)kNB ? b : (uint32_t)(kNB - 1);
  };
  const uint32_t *hcnt = hist_in ? hist_in : hc;
  if (bins && !hist_in) {  // count the outliers into key bins (the fused kernel counts while streaming)
    for (int i = tid; i < kNB; i += kThreads) hc[i] = 0u;
    tsync();
    for (int i0 = 0; i0 < (int)n_c; i0 += 4 * kThreads) {
      uint32_t b4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i = i0 + tid + j * kThreads;
        b4[j] = i < (int)n_c ? x_bits((uint32_t)i) : 0u;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (i0 + tid + j * kThreads < (int)n_c) atomicAdd(&hc[bin_of(key_of_bits(b4[j]))], 1u);
    }
    tsync();
  }
  QRITA_TSTAMP(2);

  uint32_t Kf = 0u, cutf = kNoCut, kept = (uint32_t)V;
  bool k_used_x = false;  // the final kept set is a subset of X
  bool full_row = false;
  bool sorted_out = false;  // the kept set is db/di[0, kept) (bin-sort resolve)

  // ================= bin-sort resolve (pipeline.py:199-239 on a sigma hit) =================
  // The kept set of the oracle (oracle.py:70-89) is a prefix of the (value desc, index asc) order, so
  // sort the few candidates that can be in it and take prefixes: top-k is the first k, top-p the
  // shortest prefix of the top-k whose exactly-summed renormalised mass reaches p.
  if (bins) {
    const uint32_t k = (uint32_t)pl.k;
    const bool topkp = mode == MODE_TOPKP;
    // 1. bin starts in descending order; the bin holding the k-th largest key.  A bin takes part
    //    (b >= b*) iff it starts before position k; one that is too large to order in place bails out
    //    to the pivot search before anything is overwritten.
    if (tid == 0) { sm.bail = 0u; sm.L = k; }
    uint32_t c4[4], loc = 0u;
#pragma unroll
    for (int j = 0; j < 4; ++j) { c4[j] = hcnt[kNB - 1 - 4 * tid - j]; loc += c4[j]; }
    uint32_t tot;
    uint32_t run = block_exscan_u32(loc, sm.scan_u, tot);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int b = kNB - 1 - 4 * tid - j;
      he[b] = run;
      if (run < k && k <= run + c4[j]) { sm.bstar = (uint32_t)b; sm.nabove = run; }
      if (run < k && c4[j] > (uint32_t)kMaxBin) sm.bail = 1u;
      run += c4[j];
    }
    tsync();
    QRITA_TSTAMP(10);
    const uint32_t bstar = sm.bstar;
    const uint32_t nC = sm.nabove + hcnt[bstar];
    if (nC <= (uint32_t)kCapC && sm.bail == 0u) {  // block-uniform
      // 2. counting sort by bin (bins >= b*); order inside a bin is arbitrary so far
      for (int i0 = 0; i0 < (int)n_c; i0 += 4 * kThreads) {
        uint32_t b4[4], p4[4];
        bool in4[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = i0 + tid + j * kThreads;
          b4[j] = i < (int)n_c ? x_bits((uint32_t)i) : 0u;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t bin = bin_of(key_of_bits(b4[j]));
          in4[j] = i0 + tid + j * kThreads < (int)n_c && bin >= bstar;
          p4[j] = in4[j] ? atomicAdd(&he[bin], 1u) : 0u;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (in4[j]) { cb[p4[j]] = b4[j]; ci[p4[j]] = x_idx((uint32_t)(i0 + tid + j * kThreads)); }
      }
      tsync();
      QRITA_TSTAMP(11);
      // 3. order inside every bin by (key desc, index asc), ranking against the bin's other entries;
      //    the k survivors' exp(z - max) go to ev (X is no longer needed) with per-warp exact partial
      //    sums, so the normaliser needs no pass of its own
      double *ev2 = reinterpret_cast<double *>(xb);
      Fx se = fx_zero();
      for (int q = tid; q < (int)nC; q += kThreads) {
        const uint32_t b = cb[q], ix = ci[q], key = key_of_bits(b);
        const uint32_t bin = bin_of(key);
        const uint32_t e = he[bin], c = hcnt[bin];
        uint32_t r = 0u;
#pragma unroll 4
        for (uint32_t j = e - c; j < e; ++j) {
          const uint32_t kj = key_of_bits(cb[j]);
          r += (kj > key || (kj == key && ci[j] < ix)) ? 1u : 0u;
        }
        const uint32_t d = e - c + r;
        db[d] = b; di[d] = ix;
        if (topkp && d < k) {
          const double ex = exp((double)__uint_as_float(b) - m);
          ev2[d] = ex;
          se = fx_add(se, fx_from_double(ex));
        }
      }
      if (topkp) {
        uint32_t pc[12];
        fx_split(se, pc);
#pragma unroll
        for (int i = 0; i < 12; ++i) {
          const uint32_t t = warp_sum(pc[i]);
          if (lane == 0) sm.red[0][warp][i] = t;
        }
      }
      tsync();
      QRITA_TSTAMP(12);
      {
        uint32_t L = k;
        if (topkp) {
          // 4. normaliser over the k survivors (oracle.py:85-86): exact sum, rounded once.  Lane i < 12
          //    totals piece i over the warps; the pieces are then broadcast within the warp.
          uint32_t t = 0u;
          if (lane < 12) {
#pragma unroll
            for (int w = 0; w < kWarps; ++w) t += sm.red[0][w][lane];
          }
          uint32_t pc[12];
#pragma unroll
          for (int i = 0; i < 12; ++i) pc[i] = __shfl_sync(0xffffffffu, t, i);
          const double D = fx_to_double(fx_join(pc));
          QRITA_TSTAMP(13);
          // 5. exact prefix masses in sorted order; the first prefix whose fsum reaches p
          const int E = ((int)k + kThreads - 1) / kThreads;
          const int q0 = tid * E;
          Fx sp_loc = fx_zero();
          for (int j = 0; j < E; ++j) {
            const int q = q0 + j;
            if (q < (int)k) {
              const double pi = ev2[q] / D;
              ev2[q] = pi;
              sp_loc = fx_add(sp_loc, fx_from_double(pi));
            }
          }
          Fx Mtot;
          Fx pre = block_exscan_fx(sp_loc, sm.scan_f[1], Mtot);
          QRITA_TSTAMP(14);
          for (int j = 0; j < E; ++j) {
            const int q = q0 + j;
            if (q < (int)k) {
              pre = fx_add(pre, fx_from_double(ev2[q]));
              if (fx_ge(pre, pl.t_p)) { atomicMin(&sm.L, (uint32_t)q + 1u); break; }
            }
          }
          tsync();
          // p >= fsum(all survivors): keep them all (oracle.py:45-46)
          L = fx_ge(Mtot, pl.t_sp) ? sm.L : k;
          met.p_search_iters = 1;
        }
        met.k_search_iters = 1;
        met.trunc_hit = 1;
        met.fallback_used = 0;
        Kf = key_of_bits(db[L - 1u]);
        cutf = di[L - 1u];
        kept = L;
        k_used_x = true;
        sorted_out = true;
      }
    }
    tsync();
  }
  QRITA_TSTAMP(3);
  const SrcX X{xb, xi, (int)n_c};
  const SrcRow<T> RW{in, V};
  const bool row_vec = ((uintptr_t)in % 16) == 0 && V % Vec<T>::W == 0;
  Red red(sm);
  // c-th copy of key K in index order (the duplicate-trimming rule of pipeline.py:53-56)
  auto row_select = [&](uint32_t K, uint32_t c) -> uint32_t {
    if (row_vec) {  // block counts in the first 8 KB of the work area (free whenever a cut is selected)
      bool ok;
      const uint32_t r = select_nth_eq_row<T>(in, V, K, c, sm, reinterpret_cast<uint32_t *>(work),
                                              2 * kNB, ok);
      if (ok) return r;
    }
    return select_nth_eq(RW, K, c, red);
  };
  red.act_key = (uint32_t *)ap;  // the top-k search runs first: the whole region holds keys
  red.act_pi = ap;
  red.act_cap_k = 3 * kCapA;
  red.act_cap_p = kCapA;
  red.hms = (unsigned long long *)ap;               // 5 * kBins * 8 B = 10 KB
  red.hcnt = (uint32_t *)(red.hms + 5 * kBins);     // + 1 KB  (region: 12 KB)

  // ================= top-k stage: _topk_plan, pipeline.py:88-119 =================
  uint32_t Kk = 0u, cutk = kNoCut, n_s = (uint32_t)V;  // S = {key > Kk} U {key == Kk, idx <= cutk}
  if (!sorted_out && (mode == MODE_TOPK || mode == MODE_TOPKP)) {
    const uint32_t k = (uint32_t)pl.k;
    const bool hit_ref = sigma && n_c > k;  // is_hit, sigma_trunc.py:127-133
    met.trunc_hit = (hit_ref && !force_fb) ? 1 : 0;
    met.fallback_used = met.trunc_hit ? 0 : 1;
    k_used_x = met.trunc_hit && x_fits;
    KRes kr;
    if (k_used_x) {
      kr = search_k<NP>(X, pl.key_thr ? pl.key_thr - 1u : 0u, maxkey, n_c, 0u, k, red);
    } else {
      kr = search_k<NP>(RW, lo_row, maxkey, (uint32_t)V, 0u, k, red);
      full_row = true;
    }
    met.k_search_iters = kr.iters;
    QRITA_TSTAMP(3);
    Kk = kr.K;
    uint32_t ck = k - kr.n_gt;  // n_keep = n_dup - (N - k), pipeline.py:117
    if (nodup) ck = kr.n_eq;
    if (ck >= kr.n_eq) cutk = kNoCut;
    else cutk = row_select(Kk, ck);  // index order: scan the row itself
    n_s = kr.n_gt + ck;
    Kf = Kk; cutf = cutk; kept = n_s;
    QRITA_TSTAMP(4);
  }

  // ================= top-p stage: pipeline.py:161-196 (p only) and :226-239 (k then p) ============
  bool x_ok = true;  // X still holds the outliers
  // ================= top-p only over the whole row: distinct-value path =================
  if (!sorted_out && mode == MODE_TOPP && NP == 3 && !nodup && (!x_fits || sizeof(T) == 2)) {
    // table in X (2 x 4096 words); the kCapC probabilities behind the bin-sort layout when the work
    // area has room (fused kernel: the 60 KB ring), else behind the table (staged: 64 KB X)
    constexpr uint32_t cap = 4096u;
    double *dev_pi = work_bytes >= (size_t)kWorkBytesBins + (size_t)kCapC * 8
                         ? reinterpret_cast<double *>(work + kWorkBytesBins)
                         : reinterpret_cast<double *>(xb + 2 * cap);
    const DistinctRes dr = distinct_topp<T>(P, row, in, V, m, pl, xb, xb + cap, cap, cb, ci, db, di, hc, he, dev_pi, sm);
    x_ok = false;  // the attempt used X's shared memory as its hash table
    if (dr.ok) {
      met.outlier_prob_sum = sigma ? dr.mx : 0.0;
      met.trunc_hit = (sigma && dr.hit && !force_fb) ? 1 : 0;
      met.fallback_used = met.trunc_hit ? 0 : 1;
      met.p_search_iters = 1;
      full_row = true;
      sorted_out = true;  // the stages below are done
      if (dr.keep_all) { Kf = 0u; cutf = kNoCut; kept = (uint32_t)V; }
      else {
        Kf = dr.K;
        kept = dr.n_gt + dr.j;
        cutf = dr.j >= dr.n_eq ? kNoCut : row_select(dr.K, dr.j);
      }
      QRITA_TSTAMP(13);
    }
  }
  const bool distinct_done = sorted_out && mode == MODE_TOPP;
  const bool x_fits_p = x_fits && x_ok;  // X as staged by the stream (top-p stage)

  if (!sorted_out && (mode == MODE_TOPP || mode == MODE_TOPKP)) {
    red.act_key = ak;  // (key, probability) pairs from here on
    const Fx Tp = pl.t_p, Tsp = pl.t_sp;
    const bool topp_only = (mode == MODE_TOPP);
    auto in_s = [&](uint32_t key, uint32_t idx) -> bool { return topp_only || kept_by(key, idx, Kk, cutk); };
    auto e_of = [&](uint32_t bits) -> double { return exp((double)__uint_as_float(bits) - m); };

    // ---- normaliser over the survivors (core.py:93-103; oracle.py:85-86): exact sum, rounded once
    double D;
    bool s_cached = false;
    uint32_t ns_cached = 0u;
    uint32_t cnt_dummy;
    if (!topp_only && k_used_x && n_s <= (uint32_t)kCapS) {
      // compact S into shared memory with its exp values (order is irrelevant: sums are exact)
      if (tid == 0) sm.u[4] = 0u;
      tsync();
      for (int i0 = 0; i0 < X.n; i0 += kThreads) {
        const int i = i0 + tid;
        const uint32_t b = i < X.n ? xb[i] : 0u;
        const bool in = i < X.n && kept_by(key_of_bits(b), xi[i], Kk, cutk);
        const uint32_t pos = warp_reserve(&sm.u[4], in);
        if (in) { sb[pos] = b; si[pos] = xi[i]; sp[pos] = e_of(b); }
      }
      tsync();
      ns_cached = sm.u[4];
      tsync();
      const SrcX S{sb, si, (int)ns_cached};
      const Fx Dx = block_mass(S, [&](uint32_t, uint32_t, int i, double &v) { v = sp[i]; return true; }, cnt_dummy, red);
      D = fx_to_double(Dx);
      for (int i = tid; i < (int)ns_cached; i += kThreads) sp[i] = sp[i] / D;
      tsync();
      s_cached = true;
    } else if (!topp_only && k_used_x) {
      const Fx Dx = block_mass(X, [&](uint32_t b, uint32_t ix, int, double &v) {
        if (!kept_by(key_of_bits(b), ix, Kk, cutk)) return false;
        v = e_of(b); return true; }, cnt_dummy, red);
      D = fx_to_double(Dx);
    } else {
      const Fx Dx = block_mass(RW, [&](uint32_t b, uint32_t ix, int, double &v) {
        if (!in_s(key_of_bits(b), ix)) return false;
        v = e_of(b); return true; }, cnt_dummy, red);
      D = fx_to_double(Dx);
      full_row = true;
    }
    QRITA_TSTAMP(5);
    auto pi_bits = [&](uint32_t bits) -> double { return e_of(bits) / D; };
    auto pi_key = [&](uint32_t key) -> double { return pi_bits(bits_of_key(key)); };

    // ---- pick the set the nucleus search runs on: 0 = cached S, 1 = X (filtered), 2 = full row
    int set_kind;
    uint32_t l0;
    if (topp_only) {
      // sigma hit for top-p: outlier mass > p (is_hit, sigma_trunc.py:134-138), judged exactly
      bool hit_ref = false;
      if (sigma) {
        Fx Mx;
        if (x_fits_p) {
          Mx = block_mass(X, [&](uint32_t b, uint32_t, int, double &v) { v = pi_bits(b); return true; }, cnt_dummy, red);
        } else {
          Mx = block_mass(RW, [&](uint32_t b, uint32_t, int, double &v) {
            if (key_of_bits(b) < pl.key_thr) return false;
            v = pi_bits(b); return true; }, cnt_dummy, red);
        }
        met.outlier_prob_sum = fx_to_double(Mx);
        hit_ref = fx_ge(Mx, Tsp);
      }
      met.trunc_hit = (hit_ref && !force_fb) ? 1 : 0;
      met.fallback_used = met.trunc_hit ? 0 : 1;
      if (met.trunc_hit && x_fits_p) {
        set_kind = 1; l0 = pl.key_thr ? pl.key_thr - 1u : 0u;
      } else {
        set_kind = 2; l0 = lo_row;
        full_row = true;
      }
    } else {
      set_kind = s_cached ? 0 : (k_used_x ? 1 : 2);
      l0 = Kk - 1u;  // every survivor has key >= Kk
    }

    QRITA_TSTAMP(6);
    PRes pr;
    if (set_kind == 0) {
      const SrcX S{sb, si, (int)ns_cached};
      pr = search_p<NP>(S, l0, maxkey, Tp, Tsp, [&](uint32_t, uint32_t) { return true; },
                        [&](uint32_t, int i) { return sp[i]; }, pi_key, red);
    } else if (set_kind == 1) {
      pr = search_p<NP>(X, l0, maxkey, Tp, Tsp, in_s, [&](uint32_t b, int) { return pi_bits(b); }, pi_key, red);
    } else {
      pr = search_p<NP>(RW, l0, maxkey, Tp, Tsp, in_s, [&](uint32_t b, int) { return pi_bits(b); }, pi_key, red);
    }
    if (pr.keep_all) {
      // p >= fsum(all survivors): keep them all (oracle.py:45-46)
      if (topp_only) { Kf = 0u; cutf = kNoCut; kept = (uint32_t)V; }
    } else {
      met.p_search_iters = pr.iters;
      QRITA_TSTAMP(7);
      // smallest j with fsum(head + j * p_b) >= p (_min_dup_count, pivot_search.py:143-156), exactly
      if (tid == 0) {
        const double pb = pi_key(pr.K);
        const Fx fb = fx_from_double(pb);
        const Fx need = fx_sub(Tp, pr.H);
        const double jd = ceil(fx_to_double(need) / pb);
        uint32_t j = (jd < 1.0) ? 1u : (jd > (double)pr.n_eq ? pr.n_eq : (uint32_t)jd);
        while (j > 1u && fx_ge(fx_add(pr.H, fx_mul_u32(fb, j - 1u)), Tp)) --j;
        while (j < pr.n_eq && !fx_ge(fx_add(pr.H, fx_mul_u32(fb, j)), Tp)) ++j;
        sm.u[5] = j;
      }
      tsync();
      uint32_t j = sm.u[5];
      tsync();
      if (nodup) j = pr.n_eq;
      Kf = pr.K;
      kept = pr.n_gt + j;
      if (j >= pr.n_eq) {
        // whole cluster (within S); if it is the top-k boundary cluster the top-k cut still applies
        cutf = (!topp_only && pr.K == Kk) ? cutk : kNoCut;
      } else {
        cutf = row_select(pr.K, j);  // index order: scan the row itself
      }
    }
  }

  QRITA_TSTAMP(8);
  // ================= output: finalize_mask, pipeline.py:60-78 =================
  if (mode == MODE_TOPP) {
    write_row<T>(in, out, V, Kf, cutf, inplace ? 2 : 1);  // the stream left top-p-only rows alone
  } else if (inplace) {
    write_row<T>(in, out, V, Kf, cutf, 2);
  } else if (sorted_out && !distinct_done) {
    for (int q = tid; q < (int)kept; q += kThreads) out[di[q]] = Elem<T>::from_bits(db[q]);
  } else if (k_used_x) {
    for (int i = tid; i < X.n; i += kThreads) {
      const uint32_t b = xb[i];
      if (kept_by(key_of_bits(b), xi[i], Kf, cutf)) out[xi[i]] = Elem<T>::from_bits(b);
    }
  } else {
    write_row<T>(in, out, V, Kf, cutf, 0);
  }
  QRITA_TSTAMP(9);
  if (tid == 0) {
    met.kept_count = (int32_t)kept;
    met.full_row_path = full_row ? 1 : 0;
    if (P.kept_count) P.kept_count[row] = (int32_t)kept;
    if (P.metrics) P.metrics[row] = met;
  }
}

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
// max / min / first non-finite column, order-stable outlier compaction with ballot/popc straight
// into the chunk's HBM slots, and the output background (-inf for top-k rows, a copy for
// passthrough rows).  No barriers: warps never wait for each other.
__device__ __forceinline__ float max_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float min_nan(float a, float b) {
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ bool f_nonfinite(float x) { return bits_nonfinite(__float_as_uint(x)); }

template <typename T>
__device__ __forceinline__ float lane_f(const typename Vec<T>::type &v, int w) {
  return __uint_as_float(lane_bits<T>(v, w));
}

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
    const bool write_bg = !inplace && (mode == MODE_TOPK || mode == MODE_TOPKP || mode == MODE_INVALID);
    const bool write_copy = !inplace && mode == MODE_PASS;
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
  while (*(volatile const uint32_t *)&fs.seq[slot] != g) {
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
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = (u * 32 + lane) * W;
      if (write_bg) __stcs(reinterpret_cast<VT *>(dst + e), neg_inf_vec<T>());
      else if (write_copy) __stcs(reinterpret_cast<VT *>(dst + e), v[u]);
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
  while (m) {
    const int j = __ffsll((long long)m) - 1;
    m &= m - 1;
    const int e = ((j / W) * 32 + lane) * W + (j % W);
    const uint32_t bits = Elem<T>::bits(st[e]);
    if (HIST) {
      const uint32_t bin = (key_of_bits(bits) - bl - 1u) >> bsh;
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
  const unsigned long long pol = l2_evict_first_policy();
  uint32_t g0 = 0u;  // chunks of this CTA's earlier rows: the ring's stage sequence
  for (int row = blockIdx.x; row < P.B; row += gridDim.x) {
    const T *in = (const T *)P.logits + (size_t)row * P.ld_in;
    // chunk c of the row -> stage (g0 + c) % kRing; seq records the chunk before its copy is issued
    auto issue = [&](int c) {
      const uint32_t g = g0 + (uint32_t)c, slot = g % kRing;
      *(volatile uint32_t *)&fs.seq[slot] = g;
      const uint32_t bytes = (uint32_t)(min(CE, V - c * CE) * (int)sizeof(T));
      mbar_arrive_expect_tx(&fs.full[slot], bytes);
      tma_load_1d(ring + (size_t)slot * kStageBytes, in + (size_t)c * CE, bytes, &fs.full[slot], pol);
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
      const bool hist = mode == MODE_TOPK || mode == MODE_TOPKP;
      const uint32_t bl = pl.key_thr - 1u;
      const int bsh = pl.bsh;
      const bool write_bg = !inplace && (mode == MODE_TOPK || mode == MODE_TOPKP || mode == MODE_INVALID);
      const bool write_copy = !inplace && mode == MODE_PASS;
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
                          (uint32_t)kCapXF, gxb, gxi, (uint32_t)P.xcap, fs.hist, pl.bsh,
                          (size_t)kRing * kStageBytes);
    }
    g0 += (uint32_t)nch;
    __syncthreads();  // row done: the ring and X may be refilled
  }
}

constexpr size_t kFusedDynSmem = (size_t)kCapXF * 8 + (size_t)kRing * kStageBytes;

template <typename T, int NP>
static cudaError_t launch_fused(const Params &P, cudaStream_t st) {
  static int grid_cap = 0;  // per instantiation
  if (grid_cap == 0) {
    cudaError_t e = cudaFuncSetAttribute(qrita_fused<T, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kFusedDynSmem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qrita_fused<T, NP>, kFusedThreads, kFusedDynSmem);
    if (e != cudaSuccess) return e;
    grid_cap = sms * (per_sm < 1 ? 1 : per_sm);
  }
  // Balanced persistent grid: every CTA gets the same number of rows (no partial last wave), as
  // long as that keeps >= 3/4 of the CTA slots (and their ring bytes in flight) busy.
  int grid = P.B < grid_cap ? P.B : grid_cap;
  if (P.B > grid_cap && !getenv("QRITA_UNBALANCED")) {
    const int per = (P.B + grid_cap - 1) / grid_cap;
    const int bal = (P.B + per - 1) / per;
    if (4 * bal >= 3 * grid_cap) grid = bal;
  }
  qrita_fused<T, NP><<<grid, kFusedThreads, kFusedDynSmem, st>>>(P);
  return cudaGetLastError();
}

constexpr size_t kTailDynSmem = (size_t)kCapX * 8 + (size_t)kWorkBytes;

template <typename T, int NP, bool VEC>
static cudaError_t launch_pipeline(const Params &P, cudaStream_t st, cudaEvent_t prep_done,
                                   cudaEvent_t stream_done) {
  static int stream_grid = 0;  // per instantiation
  if (stream_grid == 0) {
    cudaError_t e = cudaFuncSetAttribute(qrita_tail<T, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kTailDynSmem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qrita_stream<T, VEC>, kStreamThreads, 0);
    if (e != cudaSuccess) return e;
    // two streaming CTAs per SM leave room for one row-tail CTA, so tails run while rows stream
    int want = 3;
    if (const char *ev = getenv("QRITA_STREAM_CTAS_PER_SM")) want = atoi(ev);
    if (want < 1) want = 1;
    stream_grid = sms * (per_sm < want ? (per_sm < 1 ? 1 : per_sm) : want);
  }
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

template <typename T>
static cudaError_t launch_all(const Params &P, cudaStream_t st, bool vec, cudaEvent_t prep_done,
                              cudaEvent_t stream_done) {
  // fused single-kernel path: rows and their tail ends must be 16-byte aligned for the bulk copies
  const bool fused_ok = vec && ((size_t)P.V * sizeof(T)) % 16 == 0 && !(P.flags & QRITA_STAGED);
  if (fused_ok) {
    if (prep_done) cudaEventRecord(prep_done, st);
    cudaError_t e = (P.flags & QRITA_SEARCH_BINARY) ? launch_fused<T, 1>(P, st) : launch_fused<T, 3>(P, st);
    if (e == cudaSuccess && stream_done) e = cudaEventRecord(stream_done, st);
    return e;
  }
  if (P.flags & QRITA_SEARCH_BINARY)
    return vec ? launch_pipeline<T, 1, true>(P, st, prep_done, stream_done)
               : launch_pipeline<T, 1, false>(P, st, prep_done, stream_done);
  return vec ? launch_pipeline<T, 3, true>(P, st, prep_done, stream_done)
             : launch_pipeline<T, 3, false>(P, st, prep_done, stream_done);
}

}  // namespace qrita
