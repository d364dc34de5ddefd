// qrita_topp16.cuh — top-p-only rows of bf16 logits (cfg3: k == V, p < 1; oracle.py:57-67,
// pipeline.py:161-196) on two-CTA clusters with direct-mapped order-key histograms.
//
// A bf16 value has 65536 bit patterns, so its order key (qrita_device.cuh) shifted right by 16 is a
// 16-bit "u" that orders values exactly like the oracle's stable sort.  Each row is split into two
// contiguous segments, one per CTA of a cluster (one CTA per SM: 128 KB of shared memory hold 65536
// 16-bit counters); the row is read twice, nothing else:
//   count     every element of the segment adds 1 to counter[u] (shared atomics, no hashing, no
//             probing); row max / non-finite / 16-bit overflow are tracked on the side
//   merge     CTA q owns the u range [q * 32768, (q + 1) * 32768): the merged counts of its range
//             are the two CTAs' counters added through distributed shared memory
//   softmax   m = max u, D = sum count(u) * exp(v(u) - m) exactly (192-bit fixed point over both
//             CTAs), rounded once; pi(u) = fl(exp(v(u) - m) / D) — the same arithmetic as the single-
//             CTA distinct-value path, so the answers are bit-identical
//   nucleus   exact masses count(u) * pi(u) suffix-scanned in descending u over the cluster; the
//             boundary u = b is where the exact prefix mass crosses T(p), j* = min j with
//             S(b) + j * pi(b) >= T(p) (pivot_search.py:143-156); keep-all when fsum(all) <= p
//   output    entries with u > b, and the first j* copies of b in index order (segment 0 first:
//             its copies of b come first in the row), -inf elsewhere; or the kept-column list
// Rows the histogram cannot take (a value repeated > 65535 times in a segment, non-finite logits)
// are marked not handled and left to the fused kernel, which runs next on the same stream.
#pragma once
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "qrita_plan.cuh"


#ifndef QRITA_T16_KD  // 256-element steps of the count pass in flight per warp
#define QRITA_T16_KD 4
#endif

namespace qrita {

namespace cg = cooperative_groups;

constexpr int kT16 = 1024;                 // threads per CTA
constexpr int kW16 = kT16 / 32;
constexpr int kHistWords16 = 32768;        // 65536 16-bit counters
constexpr int kSteps16 = 2048;              // 32-value steps of the u range (1024 per CTA)
constexpr int kMaxSteps16 = 512;           // present steps per CTA range with merged counts cached
// dynamic shared memory: counters | (plan scratch, then the merged counts of the present steps) |
// step masses | present-step list
constexpr size_t kCntBytes16 = (size_t)kMaxSteps16 * 32 * 4;
constexpr size_t kTopp16DynSmem = (size_t)kHistWords16 * 4 +
                                  (sizeof(PlanScratch) > kCntBytes16 ? sizeof(PlanScratch) : kCntBytes16) +
                                  (size_t)kMaxSteps16 * sizeof(Fx) + (size_t)kMaxSteps16 * sizeof(uint16_t);

struct T16Shared {
  RowPlan pl;
  Fx wfx[kW16], wafter[kW16];
  Fx tp, tsp;                    // fixed-point thresholds of p and succ(p)
  uint32_t wu[kW16], wv[kW16], ww[kW16];
  // read by the peer CTA through distributed shared memory
  uint32_t umax, nfc, ovf;
  Fx dpart, mpart, opart;        // normaliser / mass of this CTA's u range / outlier mass
  uint32_t ocnt;                 // outliers (metrics) in this CTA's u range
  uint32_t has_cross, b, jstar, c0;  // crossing value, copies kept, its copies in segment 0
  uint32_t kq;                   // entries kept in this CTA's segment
  uint32_t pres[kSteps16 / 32];  // steps (32 consecutive u) with a value in this CTA's segment
  uint32_t nsteps, xstep;        // present steps of this CTA's u range; the step holding the crossing
};

__device__ __forceinline__ uint32_t u_full_key(uint32_t u) {
  return (u << 16) | ((u & 0x8000u) ? 0u : 0xffffu);  // positive keys: bits | 2^31; negative: ~bits
}

__device__ __forceinline__ Fx shfl_fx(const Fx &a, int src) {
  return Fx{__shfl_sync(0xffffffffu, a.w0, src), __shfl_sync(0xffffffffu, a.w1, src),
            __shfl_sync(0xffffffffu, a.w2, src)};
}

__device__ __forceinline__ Fx shfl_down_fx(const Fx &a, int d) {
  return Fx{__shfl_down_sync(0xffffffffu, a.w0, d), __shfl_down_sync(0xffffffffu, a.w1, d),
            __shfl_down_sync(0xffffffffu, a.w2, d)};
}

// exact pi(u) = fl(exp(v(u) - m) / D) — the distinct-value path's arithmetic (qrita_resolve.cuh)
__device__ __forceinline__ double pi_of_u(uint32_t u, double m, double D) {
  return exp(value_of_key(u_full_key(u)) - m) / D;
}

// QRITA_DEBUG_TIMING: %globaltimer stamps of the cluster's CTA 0 in P.dbg[row][0..6]
__device__ __forceinline__ void t16_stamp(const Params &P, int row, uint32_t q, int i) {
  if ((P.flags & QRITA_DEBUG_TIMING) && q == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    P.dbg[(size_t)row * 16 + i] = t;
  }
}

// Counters are indexed by the raw bf16 bit pattern h (no key arithmetic while counting); u is the
// order index of a value (the order key >> 16).  Both halves of the pattern space map to contiguous
// u ranges (h -> u = h ^ 0x8000 for positive, h ^ 0xffff for negative values), so 32-aligned blocks
// ("steps") of h and of u correspond.  -0.0 (h = 0x8000) ranks with +0.0 (u = 0x8000).
__device__ __forceinline__ uint32_t h_of_u(uint32_t u) { return u >= 0x8000u ? (u ^ 0x8000u) : (u ^ 0xffffu); }
__device__ __forceinline__ uint32_t u_of_h(uint32_t h) { return h < 0x8000u ? (h | 0x8000u) : (h ^ 0xffffu); }
// Counter slot of pattern h: the low 5 bits are XOR-ed with the next 5, a bijection inside every
// 32-pattern step that spreads values with zero low mantissa bits (quantised logits: 0.25, 0.5, ...)
// over the shared-memory banks instead of piling them onto bank 0.
__device__ __forceinline__ uint32_t hidx(uint32_t h) { return h ^ ((h >> 5) & 31u); }
__device__ __forceinline__ uint32_t cnt16(const uint32_t *hw, uint32_t h) {
  const uint32_t x = hidx(h);
  return (hw[x >> 1] >> ((x & 1u) << 4)) & 0xffffu;
}
__device__ __forceinline__ void hist_add(uint32_t *hw, uint32_t h, uint32_t c) {
  const uint32_t x = hidx(h);
  atomicAdd(&hw[x >> 1], c << ((x & 1u) << 4));  // result unused: red
}
// copies of value u counted in one CTA's counters
__device__ __forceinline__ uint32_t count_u(const uint32_t *hw, uint32_t u) {
  if (u == 0x8000u) return cnt16(hw, 0u) + cnt16(hw, 0x8000u);  // +0.0 and -0.0
  if (u == 0x7fffu) return 0u;                                  // (where -0.0 would map)
  return cnt16(hw, h_of_u(u));
}

static __global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kT16, 1) qrita_topp16(Params P) {
  extern __shared__ __align__(16) uint32_t hist[];
  PlanScratch *psc = reinterpret_cast<PlanScratch *>(hist + kHistWords16);
  uint32_t *cnts = hist + kHistWords16;  // aliases the plan scratch once the plan is done: [step][32]
  Fx *smass = reinterpret_cast<Fx *>(reinterpret_cast<uint8_t *>(cnts) +
                                     (sizeof(PlanScratch) > kCntBytes16 ? sizeof(PlanScratch) : kCntBytes16));
  uint16_t *steps = reinterpret_cast<uint16_t *>(smass + kMaxSteps16);
  __shared__ T16Shared s;
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t q = cl.block_rank();
  const int row = (int)(blockIdx.x >> 1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int V = P.V;
  if (row_mode(P.k[row], P.p[row], V) != MODE_TOPP) {  // uniform over the cluster: no DSMEM use
    if (q == 0 && tid == 0) P.handled[row] = 0;
    return;
  }
  const uint16_t *in = (const uint16_t *)P.logits + (size_t)row * P.ld_in;
  const int L = ((V + 1) / 2 + 7) & ~7;
  const int lo = q ? min(L, V) : 0, hi = q ? V : min(L, V);
  const bool vec = (((uintptr_t)in) & 15u) == 0;
  T16Shared *peer = cl.map_shared_rank(&s, q ^ 1u);
  const uint32_t *peer_hist = cl.map_shared_rank(hist, q ^ 1u);

  t16_stamp(P, row, q, 0);
  // (0) zero the counters and the presence map; CTA 0 plans the sigma pre-filter (metrics only)
  for (int i = tid; i < kHistWords16 / 4; i += kT16) reinterpret_cast<uint4 *>(hist)[i] = make_uint4(0, 0, 0, 0);
  if (tid < kSteps16 / 32) s.pres[tid] = 0u;
  if (tid == 0) {
    s.has_cross = 0u;
    s.tp = fx_round_threshold(P.p[row]);
    s.tsp = fx_round_threshold(nextafter(P.p[row], 2.0));
  }
  __syncthreads();
  // the sigma plan feeds only the metrics of a top-p-only row (the kept set does not depend on it)
  if (q == 0 && P.metrics && warp < kThreads / 32) {  // warps 0-7: plan_sample uses the 256-thread tsync
    if (tid == 0) plan_begin(P, row, &s.pl);
    tsync();
    plan_sample<uint16_t>(P, [&](int i) -> float { return __uint_as_float(((uint32_t)in[i]) << 16); }, in, *psc,
                          &s.pl);
  }
  if (q == 0 && !P.metrics && tid == 0) {  // status words (plan_begin writes them otherwise)
    P.status[row] = 0;
    P.nf_col[row] = -1;
    s.pl.has_thr = 0;
  }

  // (1) count pass: warp w takes the contiguous piece [lo + w * piece, ...) of the segment (the output
  //     pass's partition) in 256-element steps, one 16-byte load per lane, kD steps in flight
  const int seg = hi - lo;
  const int piece = (((seg + kW16 - 1) / kW16) + 255) & ~255;  // per warp, a multiple of 256
  const int w0 = lo + warp * piece, w1 = min(hi, w0 + piece);
  {
    auto load = [&](int e0, uint4 &w) -> int {
      const int n = max(0, min(8, w1 - e0));
      if (vec && n == 8) {
        w = *reinterpret_cast<const uint4 *>(in + e0);
      } else {
        uint32_t t[4] = {0u, 0u, 0u, 0u};
        for (int j = 0; j < n; ++j) t[j >> 1] |= ((uint32_t)in[e0 + j]) << ((j & 1) << 4);
        w = make_uint4(t[0], t[1], t[2], t[3]);
      }
      return n;
    };
    auto count8 = [&](const uint4 &c, int n) {
      const uint32_t w4[4] = {c.x, c.y, c.z, c.w};
      if (n == 8) {
#pragma unroll
        for (int j = 0; j < 4; ++j) { hist_add(hist, w4[j] & 0xffffu, 1u); hist_add(hist, w4[j] >> 16, 1u); }
      } else {
        for (int j = 0; j < n; ++j) hist_add(hist, (w4[j >> 1] >> ((j & 1) << 4)) & 0xffffu, 1u);
      }
    };
    constexpr int kD = QRITA_T16_KD;
    uint4 buf[kD];
    int nb[kD];
#pragma unroll
    for (int d = 0; d < kD; ++d) nb[d] = load(w0 + 256 * d + lane * 8, buf[d]);
    for (int e = w0 + lane * 8; e < w1 + lane * 8; e += 256 * kD) {
#pragma unroll
      for (int d = 0; d < kD; ++d) {
        const uint4 c = buf[d];
        const int n = nb[d];
        nb[d] = load(e + 256 * (d + kD), buf[d]);
        count8(c, n);
      }
    }
  }
  __syncthreads();  // every count is in
  // presence of the 32-value u steps (thread t: h steps 2t, 2t+1), the 16-bit wrap check (a wrapped
  // counter makes the sum fall short of the segment length), non-finite values (exponent 0xff)
  {
    const uint4 *hw = reinterpret_cast<const uint4 *>(hist) + tid * 8;
    uint32_t sum = 0u, nf = 0u;
#pragma unroll
    for (int hs = 0; hs < 2; ++hs) {
      uint32_t any = 0u;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint4 w = hw[hs * 4 + j];
        any |= w.x | w.y | w.z | w.w;
        sum += (w.x & 0xffffu) + (w.x >> 16) + (w.y & 0xffffu) + (w.y >> 16) + (w.z & 0xffffu) + (w.z >> 16) +
               (w.w & 0xffffu) + (w.w >> 16);
      }
      const uint32_t hstep = 2u * (uint32_t)tid + (uint32_t)hs;   // h in [32 hstep, 32 hstep + 32)
      if (any) {
        const uint32_t us = hstep < 1024u ? hstep + 1024u : hstep ^ 2047u;
        atomicOr(&s.pres[us >> 5], 1u << (us & 31u));
        if ((hstep & 1023u) >= 1020u) nf = 1u;  // h & 0x7f80 == 0x7f80: NaN / inf patterns
      }
    }
    if (tid == 512 && cnt16(hist, 0x8000u)) atomicOr(&s.pres[1024u >> 5], 1u << (1024u & 31u));  // -0.0
    sum = __reduce_add_sync(0xffffffffu, sum);
    nf = __reduce_or_sync(0xffffffffu, nf);
    if (lane == 0) { s.wu[warp] = sum; s.wv[warp] = nf; }
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t c = 0u, f = 0u;
    for (int w = 0; w < kW16; ++w) { c += s.wu[w]; f |= s.wv[w]; }
    s.ovf = c != (uint32_t)(hi - lo) ? 1u : 0u;
    s.nfc = f;
  }
  if (warp == 1) {  // this segment's largest value u (its highest present step, then the lane)
    const uint32_t lw = s.pres[lane], hw = s.pres[lane + 32];
    const unsigned hb = __ballot_sync(0xffffffffu, hw != 0u), lb = __ballot_sync(0xffffffffu, lw != 0u);
    const int wi = hb ? 32 + (31 - __clz(hb)) : 31 - __clz(lb);
    const uint32_t word = __shfl_sync(0xffffffffu, wi >= 32 ? hw : lw, wi & 31);
    const uint32_t top = (uint32_t)wi * 32u + 31u - (uint32_t)__clz(word);
    const unsigned nzl = __ballot_sync(0xffffffffu, count_u(hist, top * 32u + (uint32_t)lane) != 0u);
    if (lane == 0) s.umax = (hb | lb) ? top * 32u + 31u - (uint32_t)__clz(nzl) : 0u;
  }
  t16_stamp(P, row, q, 1);
  cl.sync();  // #1: counters, presence and the plan of both CTAs are complete
  t16_stamp(P, row, q, 2);
  if (s.nfc | peer->nfc | s.ovf | peer->ovf) {
    // non-finite logits (the fused kernel reports them) or a counter overflow: not handled here
    if (q == 0 && tid == 0) P.handled[row] = 0;
    cl.sync();  // the peer has read this CTA's scalars
    return;
  }
  const RowPlan *pl0 = q == 0 ? &s.pl : &peer->pl;
  const bool has_thr = pl0->has_thr != 0;
  const uint32_t key_thr = pl0->key_thr;
  const double p = P.p[row];
  const bool nodup = (P.flags & QRITA_NO_DUP) != 0;

  // (2) row max; this CTA's present u steps (present in either segment); their merged counts,
  //     gathered once from both CTAs' counters (one round trip of distributed shared memory)
  const uint32_t um = max(s.umax, peer->umax);
  if (warp == 0) {
    const uint32_t w0u = s.pres[lane] | peer->pres[lane], w1u = s.pres[lane + 32] | peer->pres[lane + 32];
    const uint32_t wq = q ? w1u : w0u;
    const uint32_t n = (uint32_t)__popc(wq);
    uint32_t incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    // both CTAs see both ranges' step counts: they agree on giving the row back when one overflows
    const uint32_t nother = __reduce_add_sync(0xffffffffu, (uint32_t)__popc(q ? w0u : w1u));
    const uint32_t nmine = __shfl_sync(0xffffffffu, incl, 31);
    uint32_t pos = incl - n;
    if (nmine <= (uint32_t)kMaxSteps16)
      for (uint32_t w = wq; w; w &= w - 1u) steps[pos++] = (uint16_t)(lane * 32 + __ffs(w) - 1);
    if (lane == 0) s.nsteps = (nmine > (uint32_t)kMaxSteps16 || nother > (uint32_t)kMaxSteps16) ? 0xffffffffu : nmine;
  }
  __syncthreads();
  if (s.nsteps == 0xffffffffu) {  // too many distinct values for the cached counts: fused kernel
    if (q == 0 && tid == 0) P.handled[row] = 0;
    cl.sync();
    return;
  }
  const int nst = (int)s.nsteps;
  const uint32_t ubase = q * 32768u;  // first u of this CTA's range
  for (int i = tid; i < nst * 32; i += kT16) {
    const uint32_t u = ubase + 32u * steps[i >> 5] + (uint32_t)(i & 31);
    cnts[i] = count_u(hist, u) + count_u(peer_hist, u);
  }
  __syncthreads();
  const double m = value_of_key(u_full_key(um));
  // (3) normaliser part and outlier count of the range (warps take present steps round-robin)
  {
    Fx d = fx_zero();
    uint32_t oc = 0u;
    for (int j = warp; j < nst; j += kW16) {
      const uint32_t u = ubase + 32u * steps[j] + (uint32_t)lane;
      const uint32_t c = cnts[j * 32 + lane];
      if (c) {
        d = fx_add(d, fx_mul_u32(fx_from_double(exp(value_of_key(u_full_key(u)) - m)), c));
        if (has_thr && u_full_key(u) >= key_thr) oc += c;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) d = fx_add(d, shfl_down_fx(d, o));
    oc = __reduce_add_sync(0xffffffffu, oc);
    if (lane == 0) { s.wfx[warp] = d; s.wu[warp] = oc; }
    __syncthreads();
    if (tid == 0) {
      Fx t = fx_zero();
      uint32_t c = 0u;
      for (int w = 0; w < kW16; ++w) { t = fx_add(t, s.wfx[w]); c += s.wu[w]; }
      s.dpart = t;
      s.ocnt = c;
    }
  }
  cl.sync();  // #2
  t16_stamp(P, row, q, 3);
  const double D = fx_to_double(fx_add(s.dpart, peer->dpart));
  bool keep_all = false;
  // (4) exact masses per present step; outlier mass
  {
    Fx om = fx_zero();
    for (int j = warp; j < nst; j += kW16) {
      const uint32_t u = ubase + 32u * steps[j] + (uint32_t)lane;
      const uint32_t c = cnts[j * 32 + lane];
      Fx mass = fx_zero();
      if (c) {
        mass = fx_mul_u32(fx_from_double(pi_of_u(u, m, D)), c);
        if (has_thr && u_full_key(u) >= key_thr) om = fx_add(om, mass);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) mass = fx_add(mass, shfl_down_fx(mass, o));
      if (lane == 0) smass[j] = mass;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) om = fx_add(om, shfl_down_fx(om, o));
    if (lane == 0) s.wfx[warp] = om;
  }
  __syncthreads();
  t16_stamp(P, row, q, 7);
  // suffix sums of the step masses in descending u: thread j holds present step j (nst <= 512)
  {
    const Fx mj = tid < nst ? smass[tid] : fx_zero();
    Fx incl = mj;  // inclusive suffix within the warp
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const Fx t = shfl_down_fx(incl, o);
      if (lane + o < 32) incl = fx_add(incl, t);
    }
    if (warp == 0) {  // outlier mass of the CTA (warp partials in wfx)
      Fx o = s.wfx[lane];
#pragma unroll
      for (int d = 16; d; d >>= 1) o = fx_add(o, shfl_down_fx(o, d));
      if (lane == 0) s.opart = o;
    }
    __syncthreads();
    if (lane == 0) s.wfx[warp] = incl;  // warp totals of the step masses
    __syncthreads();
    if (warp == 0) {  // per warp: the mass of the steps held by higher warps; the CTA total
      const Fx t = s.wfx[lane];
      Fx suf = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const Fx u = shfl_down_fx(suf, o);
        if (lane + o < 32) suf = fx_add(suf, u);
      }
      s.wafter[lane] = fx_sub(suf, t);
      if (lane == 0) s.mpart = suf;
    }
    __syncthreads();
    const Fx after = s.wafter[warp];
    t16_stamp(P, row, q, 8);
    cl.sync();  // #3
    t16_stamp(P, row, q, 9);
    const Fx total = fx_add(s.mpart, peer->mpart);
    const Fx Tp = s.tp, Tsp = s.tsp;
    keep_all = !fx_ge(total, Tsp);  // fsum(all) <= p (oracle.py:44-46)
    // the present step holding the crossing: S(above) < T(p) <= S(above) + mass
    const Fx above = fx_add(fx_add(q == 0 ? peer->mpart : fx_zero(), after), fx_sub(incl, mj));
    if (!keep_all && tid < nst && !fx_ge(above, Tp) && fx_ge(fx_add(above, mj), Tp)) {
      s.xstep = (uint32_t)tid;
      s.wfx[0] = above;  // read after the barrier below (the warp totals are no longer needed)
      s.has_cross = 1u;
    }
    __syncthreads();
    t16_stamp(P, row, q, 10);
    if (s.has_cross && warp == 0) {
      const uint32_t u = ubase + 32u * steps[s.xstep] + (uint32_t)lane;
      const uint32_t c = cnts[s.xstep * 32 + lane];
      const Fx f = fx_from_double(c ? pi_of_u(u, m, D) : 0.0);
      const Fx mass = c ? fx_mul_u32(f, c) : fx_zero();
      Fx suf = mass;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const Fx t = shfl_down_fx(suf, o);
        if (lane + o < 32) suf = fx_add(suf, t);
      }
      const Fx ab = fx_add(s.wfx[0], fx_sub(suf, mass));  // mass above this lane's value
      if (c && !fx_ge(ab, Tp) && fx_ge(fx_add(ab, mass), Tp)) {
        uint32_t a = 1u, z = c;  // j* = min j with S(b) + j pi(b) >= T(p) (pivot_search.py:149-156)
        if (nodup) a = z;
        while (a < z) {
          const uint32_t mid = a + (z - a) / 2u;
          if (fx_ge(fx_add(ab, fx_mul_u32(f, mid)), Tp)) z = mid;
          else a = mid + 1u;
        }
        s.b = u;
        s.jstar = a;
        s.c0 = count_u(q == 0 ? hist : peer_hist, u);  // copies of b in segment 0
      }
    }
  }
  int32_t *kidx = P.kept_idx ? P.kept_idx + (size_t)row * P.ld_idx : nullptr;
  if (q == 0 && tid == 0) {
    // row results (CTA 0): metrics (the distinct-value path's fields), status; the kept counts are
    // added by both CTAs once their output is written
    if (P.kept_count && !kidx) P.kept_count[row] = 0;
    if (P.metrics) {
      qrita_row_metrics met;
      const bool sigma = has_thr;
      const double mx = fx_to_double(fx_add(s.opart, peer->opart));
      met.outlier_count = sigma ? (int32_t)(s.ocnt + peer->ocnt) : 0;
      met.outlier_prob_sum = sigma ? mx : 0.0;
      met.trunc_hit = (sigma && mx > p && !(P.flags & QRITA_FORCE_FALLBACK)) ? 1 : 0;
      met.fallback_used = met.trunc_hit ? 0 : 1;
      met.k_search_iters = 0;
      met.p_search_iters = 1;
      met.kept_count = 0;
      met.full_row_path = 1;
      met.row_passes = 2;  // the count pass and the output pass
      P.metrics[row] = met;
    }
    P.handled[row] = 1;
  }
  cl.sync();  // #4 (also orders CTA 0's zeroed counts before both CTAs' atomic adds)
  t16_stamp(P, row, q, 4);
  uint32_t b = 0u, jstar = 0u, quota = 0u, c_mine = 0u;
  if (!keep_all) {
    const T16Shared *src = s.has_cross ? &s : peer;
    b = src->b;
    jstar = src->jstar;
    const uint32_t c0 = src->c0;  // segment 0 comes first in the row
    c_mine = count_u(hist, b);
    quota = q == 0 ? min(jstar, c_mine) : (jstar > c0 ? min(jstar - c0, c_mine) : 0u);
  }
  // kept-column lists: CTA 1's entries start after CTA 0's, so count this segment's kept entries
  // (its values above b, plus its quota of b) from the counters first
  uint32_t kbase = 0u;
  if (kidx) {
    uint32_t kc = 0u;
    if (keep_all) {
      kc = tid == 0 ? (uint32_t)(hi - lo) : 0u;
    } else {
      const uint32_t *hw = hist + tid * 32;
      for (int j = 0; j < 32; ++j) {
        const uint32_t h = hw[j];
        if (h) {
          const uint32_t x0 = (uint32_t)(tid * 64 + 2 * j);  // counter slots -> patterns (hidx is an involution)
          kc += (u_of_h(hidx(x0)) > b ? (h & 0xffffu) : 0u) + (u_of_h(hidx(x0 + 1u)) > b ? (h >> 16) : 0u);
        }
      }
      if (tid == 0) kc += quota;
    }
    kc = __reduce_add_sync(0xffffffffu, kc);
    if (lane == 0) s.wu[warp] = kc;
    __syncthreads();
    if (tid == 0) {
      uint32_t t = 0u;
      for (int w = 0; w < kW16; ++w) t += s.wu[w];
      s.kq = t;
    }
    cl.sync();  // #5
    const uint32_t k_mine = s.kq, k_peer = peer->kq;
    if (q == 0 && tid == 0) {
      if (P.kept_count) P.kept_count[row] = (int32_t)(k_mine + k_peer);
      if (P.metrics) P.metrics[row].kept_count = (int32_t)(k_mine + k_peer);
    }
    kbase = q == 0 ? 0u : k_peer;
  }
  t16_stamp(P, row, q, 5);
  t16_stamp(P, row, q ^ 1u, 12);  // CTA 1's output start / end
  // no distributed shared memory access after this point: arrive now, wait before exiting
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");

  // (5) output pass.  Warp w writes the contiguous piece [lo + w * piece, ...) of the segment in
  //     256-element steps; values compare as bf16 pairs against v(b) (IEEE: -0.0 == +0.0).  Copies of
  //     b need their ordinal in the segment only when some but not all of them are kept, kept-column
  //     lists need each kept entry's rank: then one counting pre-pass gives every warp its start.
  uint16_t *out = P.out ? (uint16_t *)P.out + (size_t)row * P.ld_out : nullptr;
  const bool ovec = vec && out && (((uintptr_t)out) & 15u) == 0;
  const bool need_ord = !keep_all && quota > 0u && quota < c_mine;
  const uint32_t bh = keep_all ? 0xff7fu : h_of_u(b);  // keep-all: compare against -max (all are >)
  const __nv_bfloat162 vb2 = __halves2bfloat162(__ushort_as_bfloat16((unsigned short)bh),
                                                __ushort_as_bfloat16((unsigned short)bh));
  auto load = [&](int e0, uint4 &w) -> int {
    const int n = max(0, min(8, w1 - e0));
    if (vec && n == 8) {
      w = *reinterpret_cast<const uint4 *>(in + e0);
    } else {
      uint32_t t[4] = {0u, 0u, 0u, 0u};
      for (int j = 0; j < n; ++j) t[j >> 1] |= ((uint32_t)in[e0 + j]) << ((j & 1) << 4);
      w = make_uint4(t[0], t[1], t[2], t[3]);
    }
    return n;
  };
  // per-element bit masks (bit j = element j of the 8) of "value > v(b)" and "value == v(b)"
  auto classify = [&](const uint4 &w, int n, uint32_t &gt, uint32_t &eq) {
    const uint32_t x[4] = {w.x, w.y, w.z, w.w};
    gt = 0u;
    eq = 0u;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const __nv_bfloat162 v2 = *reinterpret_cast<const __nv_bfloat162 *>(&x[j]);
      const uint32_t g = __hgt2_mask(v2, vb2), e = __heq2_mask(v2, vb2);
      gt |= ((g & 1u) | ((g >> 15) & 2u)) << (2 * j);
      eq |= ((e & 1u) | ((e >> 15) & 2u)) << (2 * j);
    }
    const uint32_t valid = n >= 8 ? 0xffu : ((1u << n) - 1u);
    gt &= valid;
    eq &= valid;
  };
  constexpr int kU16 = 4;  // 256-element steps per iteration: four 16-byte loads in flight per lane
  uint32_t ord = 0u, krank = kbase;  // this warp's first b-copy ordinal / kept rank
  if (need_ord || kidx) {
    uint32_t ne = 0u, nk = 0u;
    for (int e = w0 + lane * 8; e < w1 + lane * 8; e += 256 * kU16) {
      uint4 wv[kU16];
      int nv[kU16];
#pragma unroll
      for (int u = 0; u < kU16; ++u) {
        wv[u] = make_uint4(0u, 0u, 0u, 0u);
        nv[u] = e + 256 * u < w1 ? load(e + 256 * u, wv[u]) : 0;
      }
#pragma unroll
      for (int u = 0; u < kU16; ++u) {
        if (!kidx && nv[u] == 8) {  // copies of b only: 16-bit lane masks
          const uint32_t x[4] = {wv[u].x, wv[u].y, wv[u].z, wv[u].w};
          uint32_t c = 0u;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            c += (uint32_t)__popc(__heq2_mask(*reinterpret_cast<const __nv_bfloat162 *>(&x[j]), vb2));
          ne += c >> 4;
        } else {
          uint32_t gt, eq;
          classify(wv[u], nv[u], gt, eq);
          ne += (uint32_t)__popc(eq);
          nk += (uint32_t)__popc(gt);
        }
      }
    }
    ne = __reduce_add_sync(0xffffffffu, ne);
    nk = __reduce_add_sync(0xffffffffu, nk);
    if (lane == 0) { s.wv[warp] = ne; s.ww[warp] = nk; }
    __syncthreads();
    uint32_t eb = 0u, kb = 0u;
    for (int w = 0; w < warp; ++w) { eb += s.wv[w]; kb += s.ww[w]; }
    ord = eb;
    // kept entries before this warp's piece: those above b, plus the kept copies of b before it
    krank = kbase + kb + (need_ord ? min(eb, quota) : (quota == 0u ? 0u : eb));
  }
  uint32_t nkept = 0u;
  auto emit = [&](int e, const uint4 &w, int n) {
    uint32_t gt, eq;
    classify(w, n, gt, eq);
    uint32_t keepm;
    if (need_ord) {  // the first `quota` copies of b in the segment: warp-ranked
      const uint32_t ne = (uint32_t)__popc(eq);
      uint32_t incl = ne;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const uint32_t my = ord + incl - ne;
      ord += __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t r = quota > my ? min(quota - my, ne) : 0u;  // this lane keeps its first r copies
      uint32_t keq = eq;
      if (r < ne) {
        uint32_t t = eq;
        for (uint32_t i = 0; i < r; ++i) t &= t - 1u;   // drop the first r set bits ...
        keq = eq & ~t;                                   // ... and keep exactly those
      }
      keepm = gt | keq;
    } else {
      keepm = gt | (quota > 0u ? eq : 0u) | (keep_all ? eq : 0u);
    }
    nkept += (uint32_t)__popc(keepm);
    if (out && n > 0) {
      const uint32_t x[4] = {w.x, w.y, w.z, w.w};
      if (ovec && n == 8) {
        uint32_t o4[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t km = (((keepm >> (2 * j)) & 1u) ? 0x0000ffffu : 0u) |
                              (((keepm >> (2 * j + 1)) & 1u) ? 0xffff0000u : 0u);
          o4[j] = (x[j] & km) | (0xff80ff80u & ~km);
        }
        __stcs(reinterpret_cast<uint4 *>(out + e), make_uint4(o4[0], o4[1], o4[2], o4[3]));
      } else {
        for (int j = 0; j < n; ++j)
          out[e + j] = (keepm >> j) & 1u ? (uint16_t)(x[j >> 1] >> ((j & 1) << 4)) : (uint16_t)0xff80u;
      }
    }
    if (kidx) {
      const uint32_t nk = (uint32_t)__popc(keepm);
      uint32_t incl = nk;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      uint32_t pos = krank + incl - nk;
      krank += __shfl_sync(0xffffffffu, incl, 31);
      for (uint32_t mm = keepm; mm; mm &= mm - 1u) kidx[pos++] = e + __ffs(mm) - 1;
    }
  };
  // fast path (no kept-column list, full 16-byte vectors): 16-bit lane masks straight from the bf16
  // pair compares, the output word in one LOP3; copies of b are ranked only in the one 256-element
  // step of the warp where the quota runs out
  const bool fast = ovec && !kidx;
  auto emit_vec = [&](int e, const uint4 &w) {
    const uint32_t x[4] = {w.x, w.y, w.z, w.w};
    uint32_t gm[4], em[4], km[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const __nv_bfloat162 v2 = *reinterpret_cast<const __nv_bfloat162 *>(&x[j]);
      gm[j] = __hgt2_mask(v2, vb2);
      em[j] = __heq2_mask(v2, vb2);
    }
    if (keep_all) {
#pragma unroll
      for (int j = 0; j < 4; ++j) km[j] = 0xffffffffu;
    } else if (!need_ord) {
#pragma unroll
      for (int j = 0; j < 4; ++j) km[j] = gm[j] | (quota > 0u ? em[j] : 0u);
    } else {
      uint32_t ne = 0u;
#pragma unroll
      for (int j = 0; j < 4; ++j) ne += (uint32_t)__popc(em[j]);
      ne >>= 4;
      const uint32_t tot = __reduce_add_sync(0xffffffffu, ne);
      uint32_t r;  // copies of b this lane keeps
      if (ord + tot <= quota) {
        r = ne;
      } else if (ord >= quota) {
        r = 0u;
      } else {
        uint32_t incl = ne;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const uint32_t my = ord + incl - ne;
        r = quota > my ? min(quota - my, ne) : 0u;
      }
      ord += tot;
      uint32_t left = r;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t k = gm[j];
        if (r == ne) {
          k |= em[j];
        } else if (left) {  // the lane holding the quota's end: its first `left` copies
          if ((em[j] & 0xffffu) && left) { k |= 0xffffu; --left; }
          if ((em[j] & 0xffff0000u) && left) { k |= 0xffff0000u; --left; }
        }
        km[j] = k;
      }
    }
    uint32_t kc = 0u, o4[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      kc += (uint32_t)__popc(km[j]);
      o4[j] = (x[j] & km[j]) | (0xff80ff80u & ~km[j]);
    }
    nkept += kc >> 4;
    __stcs(reinterpret_cast<uint4 *>(out + e), make_uint4(o4[0], o4[1], o4[2], o4[3]));
  };
  for (int e = w0 + lane * 8; e < w1 + lane * 8; e += 256 * kU16) {
    uint4 wv[kU16];
    int nv[kU16];
#pragma unroll
    for (int u = 0; u < kU16; ++u) {
      wv[u] = make_uint4(0u, 0u, 0u, 0u);
      nv[u] = e + 256 * u < w1 ? load(e + 256 * u, wv[u]) : 0;
    }
#pragma unroll
    for (int u = 0; u < kU16; ++u) {
      if (fast && __all_sync(0xffffffffu, nv[u] == 8)) emit_vec(e + 256 * u, wv[u]);
      else emit(e + 256 * u, wv[u], nv[u]);
    }
  }
  if (!kidx) {  // kept counts: both CTAs add theirs (zeroed by CTA 0 before barrier #4)
    nkept = __reduce_add_sync(0xffffffffu, nkept);
    if (lane == 0 && nkept) {
      if (P.kept_count) atomicAdd(P.kept_count + row, (int32_t)nkept);
      if (P.metrics) atomicAdd(&P.metrics[row].kept_count, (int32_t)nkept);
    }
  }
  t16_stamp(P, row, q, 6);
  t16_stamp(P, row, q ^ 1u, 13);
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

}  // namespace qrita

namespace qrita {

static cudaError_t launch_topp16(const Params &P, cudaStream_t st) {
  static int optin[kMaxDevices] = {};
  int dummy = 0;
  cudaError_t e = per_device_once(optin, [](int, int &v) {
    v = 1;
    return cudaFuncSetAttribute(qrita_topp16, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTopp16DynSmem);
  }, dummy);
  if (e != cudaSuccess) return e;
  qrita_topp16<<<2 * P.B, kT16, kTopp16DynSmem, st>>>(P);
  return cudaGetLastError();
}


}  // namespace qrita
