// qrita_resolve.cuh — the row tail: bin-sort resolve, distinct-value top-p, full-row passes
// and tail_resolve (shared by both pipelines).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "qrita_search.cuh"

namespace qrita {

struct DistinctRes {
  bool ok;        // false: too many distinct values, use the pivot search
  bool keep_all;  // p >= fsum(all)
  uint32_t K, n_gt, n_eq, j;  // boundary key, entries above it, copies of it, copies kept
  double mx;      // outlier mass (sigma_trunc.py:121), for the hit metric
  bool hit;       // outlier mass > p
};

// Top-p over a whole row through its distinct values (pipeline.py:161-196 semantics of oracle.py:37-67).
// Equal logits have equal probabilities, so the nucleus only needs each distinct value's count: one
// pass counts them into a shared-memory hash table (batched probes; one shared atomic per
// element), then the distinct values are sorted descending (bin counting sort) and fp64 exp, the exact normaliser
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
      const uint32_t cur = *(volatile uint32_t *)&tk[h];  // (a stale read only leads to the CAS below)
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

// Kept-column list of a row (index-only output, SURVEY.md 8b kept_idx): every column with
// kept_by(key, i, K, cut) is appended to dst through a shared counter; order unspecified.  Warp-
// converged loops (uniform trip counts) so the per-warp reservation can use full-mask shuffles.
__device__ __forceinline__ uint32_t warp_reserve_n(uint32_t *ctr, uint32_t n) {
  const int lane = threadIdx.x & 31;
  uint32_t incl = n;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
  uint32_t base = 0u;
  if (lane == 0 && tot) base = atomicAdd(ctr, tot);
  return __shfl_sync(0xffffffffu, base, 0) + incl - n;
}

template <typename T>
__device__ void write_row_idx(const T *in, int V, uint32_t K, uint32_t cut, int32_t *dst, uint32_t *ctr) {
  using VT = typename Vec<T>::type;
  constexpr int W = Vec<T>::W;
  const int tid = threadIdx.x;
  if (((uintptr_t)in % 16) == 0 && V % W == 0) {
    const VT *pi = reinterpret_cast<const VT *>(in);
    const int nv = V / W;
    const VecCmp<T> cmp(K);
    for (int b0 = 0; b0 < nv; b0 += kThreads * kLd) {
      VT r[kLd];
#pragma unroll
      for (int j = 0; j < kLd; ++j)
        if (b0 + j * kThreads + tid < nv) r[j] = __ldcg(pi + b0 + j * kThreads + tid);
#pragma unroll
      for (int j = 0; j < kLd; ++j) {
        const int vi = b0 + j * kThreads + tid;
        uint32_t kp = 0u;
        if (vi < nv) {
          uint32_t gt, eq;
          cmp.masks(r[j], gt, eq);
          kp = gt;
#pragma unroll
          for (int w = 0; w < W; ++w)
            if (((eq >> w) & 1u) && (uint32_t)(vi * W + w) <= cut) kp |= 1u << w;
        }
        uint32_t pos = warp_reserve_n(ctr, (uint32_t)__popc(kp));
        while (kp) {
          const int w = __ffs(kp) - 1;
          kp &= kp - 1u;
          dst[pos++] = vi * W + w;
        }
      }
    }
    return;
  }
  for (int i0 = 0; i0 < V; i0 += kThreads) {
    const int i = i0 + tid;
    const bool kp = i < V && kept_by(key_of_bits(Elem<T>::bits(in[i])), (uint32_t)i, K, cut);
    const uint32_t pos = warp_reserve_n(ctr, kp ? 1u : 0u);
    if (kp) dst[pos] = i;
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
  if (tid == 0) sm.row_passes = 1u;  // the streaming pass; full-row re-reads below add to it
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
    if (P.kept_idx)
      for (int i = tid; i < V; i += kThreads) P.kept_idx[(size_t)row * P.ld_idx + i] = i;
    if (tid == 0) {
      met.kept_count = V;
      met.row_passes = 1;
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
      // (key, ~index) composites of the binned candidates in X's free index half: one 64-bit
      // compare per pair in the ranking below
      unsigned long long *ck = reinterpret_cast<unsigned long long *>(xi);
      for (int q = tid; q < (int)nC; q += kThreads)
        ck[q] = ((unsigned long long)key_of_bits(cb[q]) << 32) | (0xffffffffu - ci[q]);
      tsync();
      Fx se = fx_zero();
      for (int q = tid; q < (int)nC; q += kThreads) {
        const uint32_t b = cb[q], ix = ci[q], key = key_of_bits(b);
        const uint32_t bin = bin_of(key);
        const uint32_t e = he[bin], c = hcnt[bin];
        uint32_t r = 0u;
        const unsigned long long cq = ck[q];
#pragma unroll 4
        for (uint32_t j = e - c; j < e; ++j) r += ck[j] > cq ? 1u : 0u;
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
      if (ok) {
        if (tid == 0) ++sm.row_passes;
        return r;
      }
    }
    if (tid == 0) ++sm.row_passes;
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
      if (tid == 0) sm.row_passes += (uint32_t)kr.src_passes;
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
    if (tid == 0) ++sm.row_passes;  // its counting pass read the whole row
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
      if (tid == 0) ++sm.row_passes;
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
          if (tid == 0) ++sm.row_passes;
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
      if (tid == 0) sm.row_passes += (uint32_t)pr.src_passes;
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
  // kept-column list (kept_idx): the same four sources as the masked values below
  if (P.kept_idx) {
    int32_t *dst = P.kept_idx + (size_t)row * P.ld_idx;
    if (tid == 0) sm.u[6] = 0u;
    tsync();
    if (mode == MODE_TOPP || (!sorted_out && !k_used_x)) {
      if (!P.out && tid == 0) ++sm.row_passes;  // (with masked output, write_row's pass is counted below)
      write_row_idx<T>(in, V, Kf, cutf, dst, &sm.u[6]);
    } else if (sorted_out) {
      for (int q = tid; q < (int)kept; q += kThreads) dst[q] = (int32_t)di[q];
    } else {
      for (int i0 = 0; i0 < X.n; i0 += kThreads) {
        const int i = i0 + tid;
        const bool kp = i < X.n && kept_by(key_of_bits(xb[i]), xi[i], Kf, cutf);
        const uint32_t pos = warp_reserve_n(&sm.u[6], kp ? 1u : 0u);
        if (kp) dst[pos] = (int32_t)xi[i];
      }
    }
    tsync();
  }
  if (!P.out) {  // index-only call
  } else if (mode == MODE_TOPP || inplace || (!sorted_out && !k_used_x)) {
    if (tid == 0) ++sm.row_passes;  // write_row reads the whole row again
  }
  if (!P.out) {
  } else if (mode == MODE_TOPP) {
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
    met.row_passes = (int32_t)sm.row_passes;
    if (P.kept_count) P.kept_count[row] = (int32_t)kept;
    if (P.metrics) P.metrics[row] = met;
  }
}

}  // namespace qrita
