// qrita_search.cuh — block primitives of the row tail and the exact pivot searches
// (pivot_search.py:93-244) with duplicate selection.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "qrita_plan.cuh"

namespace qrita {

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
  uint32_t row_passes;          // full passes over the row's logits in this row's tail
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
  int src_passes;  // full passes over src (bracket, compaction, passes before compaction)
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
  int sp = 0;  // full passes over src
  if (r - l > (uint32_t)(4 * kBins)) {
    ++sp;
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
      ++sp;
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
      ++sp;
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
  const KRes res = st.done ? KRes{st.K, st.n_gt, st.n_eq, st.iters, sp}
                           : KRes{st.r, st.cr, st.cl - st.cr, st.iters, sp};
  tsync();
  return res;
}

struct PRes {
  int src_passes;  // full passes over src
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
  int sp = 1;  // full passes over src: the bracketing pass or the total-mass pass, then below
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
      res.src_passes = sp;
      tsync();
      return res;
    }
    tsync();  // every thread has read st.compact above
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
      res.src_passes = sp;
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
      ++sp;
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
      ++sp;
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
  const PRes res = st.done ? PRes{sp, st.K, st.n_gt, st.n_eq, st.H, st.iters, false, fx_zero()}
                           : PRes{sp, st.r, st.cr, st.cl - st.cr, st.Mr, st.iters, false, fx_zero()};
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

}  // namespace qrita
