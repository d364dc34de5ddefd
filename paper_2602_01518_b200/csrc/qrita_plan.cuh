// qrita_plan.cuh — per-row plan: the reference's sigma statistics (numpy pairwise sums),
// threshold, nucleus thresholds; the staged pipeline's qrita_prep kernel.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "qrita_elem.cuh"

namespace qrita {

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
__device__ void plan_sample(const Params &P, SampleAt xs, const T *a, PlanScratch &sc, RowPlan *out,
                            int tid_base = 0, bool leaves_done = false) {
  // tid_base: the kThreads-thread group runs from warp tid_base / 32; leaves_done: the caller already
  // filled sc.acc with the leaf loop below (the default 4096-sample perfect tree only)
  const int tid = (int)threadIdx.x - tid_base;
  if (!out->has_thr) return;  // uniform per group (written before the caller's barrier)
  const PwTree &tr = P.tree;
  const int n = tr.n;
  const int nl = tr.n_leaves;
  if (nl > 0) {
    // numpy's 8-accumulator leaf loop, one thread per (leaf, accumulator)
    for (int q = leaves_done ? nl * 8 : tid; q < nl * 8; q += kThreads) {
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

}  // namespace qrita
