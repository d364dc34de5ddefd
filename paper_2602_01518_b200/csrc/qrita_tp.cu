// qrita_tp.cu — vocab-sharded (tensor-parallel LM-head) exact Top-k / Top-p (BASELINE cfg5,
// SURVEY.md 8(b) qrita_topk_topp_tp, 8(e) "vocab-sharded: one or two exchanges").
//
// Every rank holds a contiguous column shard [B, Vr] of the [B, V] logits and produces its shard of
// the unsharded answer (pkg/src/sigmatop/oracle.py:70-89; pipeline.py:199-239), bit-exact.  Only
// per-row partials cross ranks, through a qrita_comm (NCCL, loaded at run time, or a host-staged
// exchange supplied by the caller):
//
//  top-k / top-k+top-p rows (k < V):
//    tp_prep  -> k_loc = min(k, Vr)             (top-p-only rows: k_loc = 1, i.e. the local max)
//    local top-k_loc with the single-GPU kernels (index-only output, one read of the shard)
//    tp_pack_sorted -> (order key, global column) pairs sorted by (value desc, column asc), padded
//                 to kmax per row (already in order when the shard call's bin-sort emitted them so)
//    all_gather                                   <= 8 * kmax bytes per row per rank
//    tp_merge_resolve -> the ranks' sorted lists merged (bitonic merge tree, or binary-search ranks)
//                 into the global top-k in order, then the exact normaliser / nucleus over it with
//                 the ORIGINAL k and p: the global top-k is a subset of the union of the local top-k
//                 sets, and the full-row max (the global top-1), the survivor normaliser and the
//                 nucleus all depend on that set only
//    (candidate rows wider than kSmallW: tp_pack by column, tp_merge into column-ordered rows, and
//    the single-GPU kernels on them)
//  top-p-only rows (k == V, p < 1), which need the whole row:
//    global max   = max of the gathered local maxima
//    tp_denom -> D = sum_i exp(z_i - m) as exact 192-bit fixed point, 4 limbs of 48 bits
//                 (an integer all-reduce SUM is exact and order-independent), rounded once
//    tp_pass x 8 (fp32) / x 4 (bf16): 16 thresholds per pass over the order-key interval (lo, hi]
//                 holding the nucleus boundary; per threshold (count, exact mass of pi = fl(e/D))
//                 of the keys above it -> all-reduce SUM -> the sub-interval where the exact prefix
//                 mass crosses T(p) (the smallest fixed-point mass whose fsum reaches p)
//    tp_quota -> boundary key b, S(b) = exact mass above b, j* = min j : S(b) + j * pi_b >= T(p)
//                 (pivot_search.py:143-156), and this rank's copies of b -> all-reduce of the
//                 per-rank counts; copies are kept in global index order = rank order
//  tp_write -> the shard output: -inf background, kept entries bit-identical to the input.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <float.h>
#include <stdio.h>
#include <nccl.h>
#include <stdint.h>
#include <string.h>

#include <mutex>

#include "qrita_internal.h"
#include "qrita_search.cuh"

namespace qrita {
namespace tp {

constexpr int kT = 256;             // threads per row CTA
constexpr int kR = 16;              // thresholds per radix pass (4 key bits)
constexpr int kPartWords = kR * 5;  // per row and pass: 16 x (count, 4 mass limbs of 48 bits)
constexpr int kMaxShard = 1 << 20;  // columns per shard (shared-memory column bitmap <= 128 KB)
constexpr int kMaxWorld = 1024;
constexpr unsigned long long kM48 = (1ull << 48) - 1ull;

enum RowState : int32_t { SEARCHING = 0, FOUND = 1, KEEP_ALL = 2 };

struct alignas(16) TpRow {
  Fx S_lo, S_hi;                  // exact mass of the keys > lo, > hi (top-p-only rows)
  Fx t_p, t_sp;                   // fixed-point thresholds of p and succ(p)
  unsigned long long C_lo, C_hi;  // counts of the keys > lo, > hi
  double D;                       // normaliser, the exact sum rounded once
  uint32_t lo, hi;                // radix interval (lo, hi] in key units >> sh
  uint32_t maxkey;                // global max order key
  int32_t mode;                   // MODE_* of the GLOBAL row (MODE_INVALID on bad input)
  int32_t state;                  // RowState
  uint32_t c_local;               // this shard's copies of the boundary key (last interval)
  uint32_t jstar;                 // copies of the boundary key kept over all shards
  int32_t pad;
};

// ------------------------------------------------------------------------------------------------
// small device helpers
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ void fx_to_limbs48(const Fx &a, unsigned long long *l) {
  l[0] = a.w0 & kM48;
  l[1] = ((a.w0 >> 48) | (a.w1 << 16)) & kM48;
  l[2] = ((a.w1 >> 32) | (a.w2 << 32)) & kM48;
  l[3] = a.w2 >> 16;
}

// sum of limbs (each < 2^64 after an all-reduce of <= 2^16 ranks) back to 192-bit fixed point
__device__ __forceinline__ Fx fx_from_limbs48(const unsigned long long *l) {
  Fx r{l[0], 0ull, 0ull};
  r = fx_add(r, Fx{l[1] << 48, l[1] >> 16, 0ull});
  r = fx_add(r, Fx{0ull, l[2] << 32, l[2] >> 32});
  r = fx_add(r, Fx{0ull, 0ull, l[3] << 16});
  return r;
}

__device__ __forceinline__ Fx warp_sum_fx(Fx a) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    Fx b{__shfl_xor_sync(0xffffffffu, a.w0, o), __shfl_xor_sync(0xffffffffu, a.w1, o),
         __shfl_xor_sync(0xffffffffu, a.w2, o)};
    a = fx_add(a, b);
  }
  return a;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long a) {
#pragma unroll
  for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  return a;
}

// exclusive scan over the CTA (kT threads, one value each, thread order)
__device__ __forceinline__ uint32_t cta_exscan(uint32_t v, uint32_t *buf, uint32_t &total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) buf[warp] = incl;
  __syncthreads();
  uint32_t before = 0u, tot = 0u;
#pragma unroll
  for (int w = 0; w < kT / 32; ++w) {
    before += (w < warp) ? buf[w] : 0u;
    tot += buf[w];
  }
  __syncthreads();
  total = tot;
  return before + incl - v;
}

template <typename T>
__device__ __forceinline__ uint32_t key_at(const T *row, int c) {
  return key_of_bits(Elem<T>::bits(row[c]));
}

// The order key of a bf16 value in the search's units u = key >> 16 (the low half of a bf16 key is
// 0x0000 for positive values, whose key is bits | 2^31, and 0xffff for negative ones, key = ~bits).
__device__ __forceinline__ uint32_t full_key(uint32_t u, int sh) {
  if (!sh) return u;
  return (u << 16) | ((u & 0x8000u) ? 0u : 0xffffu);
}

// thresholds of the radix pass over (lo, hi]: T_j = lo + floor(j * (hi - lo) / 16), j = 0..15
__device__ __forceinline__ uint32_t thr(uint32_t lo, uint32_t hi, int j) {
  return lo + (uint32_t)(((unsigned long long)j * (unsigned long long)(hi - lo)) >> 4);
}

// Folds the all-reduced partials of the pass that ran over (lo, hi] into the row state: the new
// interval is (T_sel, T_sel+1] with sel the largest threshold whose mass above still reaches T(p).
__device__ void tp_update(TpRow &R, const unsigned long long *part, const unsigned long long *part_loc,
                          bool first) {
  Fx S[kR];
  unsigned long long C[kR];
#pragma unroll
  for (int j = 0; j < kR; ++j) {
    S[j] = fx_add(R.S_hi, fx_from_limbs48(part + j * 5 + 1));
    C[j] = R.C_hi + part[j * 5];
  }
  if (first && !fx_ge(S[0], R.t_sp)) {  // fsum(all) <= p: the oracle keeps the whole row
    R.state = KEEP_ALL;
    return;
  }
  int sel = 0;
#pragma unroll
  for (int j = 1; j < kR; ++j)
    if (fx_ge(S[j], R.t_p)) sel = j;
  const uint32_t lo = thr(R.lo, R.hi, sel);
  const uint32_t hi = sel + 1 < kR ? thr(R.lo, R.hi, sel + 1) : R.hi;
  const unsigned long long nl_lo = part_loc[sel * 5], nl_hi = sel + 1 < kR ? part_loc[(sel + 1) * 5] : 0ull;
  R.c_local = (uint32_t)(nl_lo - nl_hi);
  if (sel + 1 < kR) {
    R.S_hi = S[sel + 1];
    R.C_hi = C[sel + 1];
  }
  R.S_lo = S[sel];
  R.C_lo = C[sel];
  R.lo = lo;
  R.hi = hi;
  if (hi - lo == 1u) R.state = FOUND;
}

// ------------------------------------------------------------------------------------------------
// kernels
// ------------------------------------------------------------------------------------------------
__global__ void tp_prep(int B, int Vg, int Vr, int kcap, int no_topp, const int64_t *k, const double *p,
                        int64_t *k_loc, double *p_one, TpRow *rows, int32_t *tst) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= B) return;
  const int64_t kk = k[r];
  const double pp = p[r];
  int mode = row_mode(kk, pp, Vg);
  int32_t st = 0;
  if (!(kk >= 1 && kk <= (int64_t)Vg)) st |= ST_BAD_K;
  if (!(pp > 0.0 && pp <= 1.0)) st |= ST_BAD_P;
  const bool topk = mode == MODE_TOPK || mode == MODE_TOPKP;
  if ((topk && kk > (int64_t)kcap) || (no_topp && mode == MODE_TOPP)) st |= ST_TP_KCAP;
  if (st) mode = MODE_INVALID;
  tst[r] = st;
  k_loc[r] = (mode == MODE_TOPK || mode == MODE_TOPKP) ? (kk < (int64_t)Vr ? kk : (int64_t)Vr) : 1;
  p_one[r] = 1.0;
  TpRow R;
  memset(&R, 0, sizeof(R));
  R.mode = mode;
  rows[r] = R;
}

// Local candidates of row blockIdx.x, in column order: kept columns -> shared bitmap -> ordered scan.
// send = [counts (B4 words) | keys [B][kmax] | global columns [B][kmax]].
template <typename T>
__global__ void __launch_bounds__(kT) tp_pack(const T *logits, int64_t ld, int Vr, int64_t offset, int kmax,
                                             const int32_t *kc, const int32_t *kidx, uint32_t *send, int B4,
                                             int B, int ordered) {
  extern __shared__ uint32_t bm[];
  __shared__ uint32_t buf[kT / 32];
  const int r = blockIdx.x, tid = threadIdx.x;
  uint32_t *keys = send + B4 + (size_t)r * kmax;
  uint32_t *gid = send + B4 + (size_t)B * kmax + (size_t)r * kmax;
  const int cnt = kc[r];
  const T *row = logits + (size_t)r * ld;
  if (!ordered) {
    // the small-row resolve orders ties by global column itself: the list order is free
    for (int i = tid; i < kmax; i += kT) {
      const int c = i < cnt ? kidx[(size_t)r * kmax + i] : 0;
      keys[i] = i < cnt ? key_at(row, c) : 0u;
      gid[i] = i < cnt ? (uint32_t)(offset + c) : 0xffffffffu;
    }
    if (tid == 0) send[r] = (uint32_t)cnt;
    return;
  }
  const int nw = (Vr + 31) >> 5;
  for (int i = tid; i < nw; i += kT) bm[i] = 0u;
  __syncthreads();
  for (int i = tid; i < cnt; i += kT) {
    const int c = kidx[(size_t)r * kmax + i];
    atomicOr(&bm[c >> 5], 1u << (c & 31));
  }
  __syncthreads();
  const int per = (nw + kT - 1) / kT;
  const int w0 = tid * per, w1 = min(nw, w0 + per);
  uint32_t mine = 0u;
  for (int w = w0; w < w1; ++w) mine += __popc(bm[w]);
  uint32_t total;
  uint32_t pos = cta_exscan(mine, buf, total);
  for (int w = w0; w < w1; ++w) {
    uint32_t m = bm[w];
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1u;
      const int c = w * 32 + b;
      keys[pos] = key_at(row, c);
      gid[pos] = (uint32_t)(offset + c);
      ++pos;
    }
  }
  for (int i = cnt + tid; i < kmax; i += kT) {
    keys[i] = 0u;
    gid[i] = 0xffffffffu;
  }
  if (tid == 0) send[r] = (uint32_t)cnt;
}

// Candidate rows in global column order (the ranks' lists concatenated), padded with -FLT_MAX at
// the end; top-p-only rows: the global max key.  Rows that are not top-k get a dummy k = 1, p = 1.
__global__ void __launch_bounds__(kT) tp_merge(const uint32_t *recv, size_t send_words, int B4, int B, int kmax,
                                              int world, int W, const int64_t *k, const double *p, TpRow *rows,
                                              float *cval, uint32_t *cgid, int64_t *k_c, double *p_c) {
  __shared__ uint32_t off[kMaxWorld + 1];
  const int r = blockIdx.x, tid = threadIdx.x;
  const int mode = rows[r].mode;
  if (tid == 0) {
    uint32_t acc = 0u, mk = 0u;
    for (int g = 0; g < world; ++g) {
      const uint32_t *sg = recv + (size_t)g * send_words;
      off[g] = acc;
      acc += sg[r];
      // top-p-only rows: each shard sent one candidate, its max
      if (sg[r]) mk = max(mk, sg[B4 + (size_t)r * kmax]);
    }
    off[world] = acc;
    if (mode == MODE_TOPP) rows[r].maxkey = mk;
  }
  __syncthreads();
  float *cv = cval + (size_t)r * W;
  uint32_t *cg = cgid + (size_t)r * W;
  const bool topk = mode == MODE_TOPK || mode == MODE_TOPKP;
  const uint32_t n = topk ? off[world] : 0u;
  if (topk) {
    for (int g = 0; g < world; ++g) {
      const uint32_t *sg = recv + (size_t)g * send_words;
      const uint32_t *keys = sg + B4 + (size_t)r * kmax;
      const uint32_t *gid = sg + B4 + (size_t)B * kmax + (size_t)r * kmax;
      const uint32_t o = off[g], ng = off[g + 1] - off[g];
      for (uint32_t i = tid; i < ng; i += kT) {
        cv[o + i] = __uint_as_float(bits_of_key(keys[i]));
        cg[o + i] = gid[i];
      }
    }
  }
  for (uint32_t i = n + tid; i < (uint32_t)W; i += kT) {
    cv[i] = -FLT_MAX;
    cg[i] = 0xffffffffu;
  }
  if (tid == 0) {
    k_c[r] = topk ? k[r] : 1;
    p_c[r] = topk ? p[r] : 1.0;
  }
}

// Exact normaliser partial of this shard (top-p-only rows): sum exp(z - m) in fixed point.
template <typename T>
__global__ void __launch_bounds__(kT) tp_denom(const T *logits, int64_t ld, int Vr, const double *p, TpRow *rows,
                                              unsigned long long *dl, int sh) {
  __shared__ Fx red[kT / 32];
  const int r = blockIdx.x, tid = threadIdx.x;
  TpRow R = rows[r];
  if (R.mode != MODE_TOPP) {
    if (tid < 4) dl[(size_t)r * 4 + tid] = 0ull;
    return;
  }
  const double m = value_of_key(R.maxkey);
  const T *row = logits + (size_t)r * ld;
  Fx acc = fx_zero();
  for (int c = tid; c < Vr; c += kT)
    acc = fx_add(acc, fx_from_double(exp((double)__uint_as_float(Elem<T>::bits(row[c])) - m)));
  acc = warp_sum_fx(acc);
  if ((tid & 31) == 0) red[tid >> 5] = acc;
  __syncthreads();
  if (tid == 0) {
    Fx s = fx_zero();
    for (int w = 0; w < kT / 32; ++w) s = fx_add(s, red[w]);
    fx_to_limbs48(s, dl + (size_t)r * 4);
    R.lo = 0u;
    R.hi = R.maxkey >> sh;
    R.S_hi = fx_zero();
    R.C_hi = 0ull;
    R.state = SEARCHING;
    R.t_p = fx_round_threshold(p[r]);
    R.t_sp = fx_round_threshold(nextafter(p[r], 2.0));
    rows[r] = R;
  }
}

// One radix pass (top-p-only rows): fold the previous pass, then per threshold T_j of the current
// interval the count and exact mass of this shard's keys in (T_j, hi].
template <typename T>
__global__ void __launch_bounds__(kT) tp_pass(const T *logits, int64_t ld, int Vr, TpRow *rows,
                                             const unsigned long long *dl, unsigned long long *part,
                                             unsigned long long *part_loc, int q, int sh) {
  __shared__ TpRow Rs;
  __shared__ Fx red_f[kR][kT / 32];
  __shared__ unsigned long long red_c[kR][kT / 32];
  const int r = blockIdx.x, tid = threadIdx.x;
  unsigned long long *pr = part + (size_t)r * kPartWords, *pl = part_loc + (size_t)r * kPartWords;
  if (tid == 0) {
    TpRow R = rows[r];
    if (R.mode == MODE_TOPP) {
      if (q == 0) {
        R.D = fx_to_double(fx_from_limbs48(dl + (size_t)r * 4));
      } else if (R.state == SEARCHING) {
        tp_update(R, pr, pl, q == 1);
      }
      rows[r] = R;
    }
    Rs = R;
  }
  __syncthreads();
  const TpRow R = Rs;
  if (R.mode != MODE_TOPP || R.state != SEARCHING) {
    for (int i = tid; i < kPartWords; i += kT) {
      pr[i] = 0ull;
      pl[i] = 0ull;
    }
    return;
  }
  __syncthreads();  // every thread has read the previous partials before they are overwritten
  uint32_t t[kR];
#pragma unroll
  for (int j = 0; j < kR; ++j) t[j] = thr(R.lo, R.hi, j);
  const double m = value_of_key(R.maxkey);
  const T *row = logits + (size_t)r * ld;
  Fx acc[kR];
  uint32_t cnt[kR];
#pragma unroll
  for (int j = 0; j < kR; ++j) {
    acc[j] = fx_zero();
    cnt[j] = 0u;
  }
  for (int c = tid; c < Vr; c += kT) {
    const uint32_t key = key_at(row, c);
    const uint32_t u = key >> sh;
    if (u > R.lo && u <= R.hi) {
      const Fx f = fx_from_double(exp(value_of_key(key) - m) / R.D);
#pragma unroll
      for (int j = 0; j < kR; ++j) {
        if (u > t[j]) {
          acc[j] = fx_add(acc[j], f);
          ++cnt[j];
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kR; ++j) {
    const Fx a = warp_sum_fx(acc[j]);
    const unsigned long long n = warp_sum_u64(cnt[j]);
    if ((tid & 31) == 0) {
      red_f[j][tid >> 5] = a;
      red_c[j][tid >> 5] = n;
    }
  }
  __syncthreads();
  if (tid < kR) {
    Fx s = fx_zero();
    unsigned long long n = 0ull;
    for (int w = 0; w < kT / 32; ++w) {
      s = fx_add(s, red_f[tid][w]);
      n += red_c[tid][w];
    }
    unsigned long long l[4];
    fx_to_limbs48(s, l);
    pr[tid * 5] = n;
    pl[tid * 5] = n;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      pr[tid * 5 + 1 + i] = l[i];
      pl[tid * 5 + 1 + i] = l[i];
    }
  }
}

// Boundary key, j* and this shard's tie count (top-p-only rows), one thread per row.
__global__ void tp_quota(int B, TpRow *rows, const unsigned long long *part, const unsigned long long *part_loc,
                         uint32_t *qbuf, int rank, int world, int sh) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= B) return;
  for (int g = 0; g < world; ++g) qbuf[(size_t)r * world + g] = 0u;
  TpRow R = rows[r];
  if (R.mode != MODE_TOPP) return;
  if (R.state == SEARCHING) tp_update(R, part + (size_t)r * kPartWords, part_loc + (size_t)r * kPartWords, false);
  if (R.state == FOUND) {
    const uint32_t b = full_key(R.hi, sh);
    const double m = value_of_key(R.maxkey);
    const Fx fb = fx_from_double(exp(value_of_key(b) - m) / R.D);
    const unsigned long long nb = R.C_lo - R.C_hi;
    uint32_t lo = 1u, hi = (uint32_t)nb;
    while (lo < hi) {
      const uint32_t mid = lo + (hi - lo) / 2u;
      if (fx_ge(fx_add(R.S_hi, fx_mul_u32(fb, mid)), R.t_p)) hi = mid;
      else lo = mid + 1u;
    }
    R.jstar = lo;
    qbuf[(size_t)r * world + rank] = R.c_local;
#ifdef QRITA_TP_DEBUG
    if (r < 2)
      printf("row %d rank %d: b %08x lo %u hi %u C_lo %llu C_hi %llu S_hi %llx:%llx:%llx t_p %llx:%llx:%llx fb %llx:%llx:%llx "
             "D %.17g j* %u c_local %u\n", r, rank, b, R.lo, R.hi, R.C_lo, R.C_hi, R.S_hi.w2, R.S_hi.w1, R.S_hi.w0,
             R.t_p.w2, R.t_p.w1, R.t_p.w0, fb.w2, fb.w1, fb.w0, R.D, R.jstar, R.c_local);
#endif
  }
  rows[r] = R;
}

// The shard output: -inf background, kept entries bit-identical; kept_count of this shard.
template <typename T>
__global__ void __launch_bounds__(kT) tp_write(const T *logits, int64_t ld_in, T *out, int64_t ld_out, int Vr,
                                              int64_t offset, const TpRow *rows, const uint32_t *cgid,
                                              const int32_t *kidx_c, const int32_t *kc_c, int W,
                                              const uint32_t *qbuf, int rank, int world, int32_t *kept_count,
                                              int32_t *status, const int32_t *tst, int sh, int bg_done,
                                              const int32_t *kidx_s, const int32_t *kc_s, int kmax,
                                              const unsigned long long *bnd, const uint32_t *send, int B4,
                                              int B) {
  extern __shared__ uint32_t bm[];
  __shared__ uint32_t buf[kT / 32];
  __shared__ uint32_t nkept;
  const int r = blockIdx.x, tid = threadIdx.x;
  const TpRow R = rows[r];
  if (tid == 0) {
    status[r] |= tst[r];
    nkept = 0u;
  }
  const T *in = logits + (size_t)r * ld_in;
  T *o = out + (size_t)r * ld_out;
  const T ninf = Elem<T>::neg_inf();
  uint32_t kept = 0u;
  if ((R.mode == MODE_TOPK || R.mode == MODE_TOPKP) && bg_done && bnd) {
    // the shard call wrote the local top-k over a -inf background; the global kept set is every
    // candidate whose (key, ~global column) composite reaches the resolve's boundary: clear the rest
    // (the rank's own sorted candidate list is in its send buffer: keys, then global columns)
    const unsigned long long bd = bnd[r];
    const int nl = kc_s[r];
    const uint32_t *keys = send + B4 + (size_t)r * kmax;
    const uint32_t *gid = send + B4 + (size_t)B * kmax + (size_t)r * kmax;
    for (int i = tid; i < nl; i += kT) {
      const uint32_t g = gid[i];
      const unsigned long long cc = ((unsigned long long)keys[i] << 32) | (0xffffffffu - g);
      if (cc >= bd) ++kept;
      else o[(int64_t)g - offset] = ninf;
    }
  } else if (R.mode == MODE_TOPK || R.mode == MODE_TOPKP) {
    const int nw = (Vr + 31) >> 5;
    for (int i = tid; i < nw; i += kT) bm[i] = 0u;
    __syncthreads();
    const int n = kc_c[r];
    for (int i = tid; i < n; i += kT) {
      const int32_t e = kidx_c[(size_t)r * W + i];
      const uint32_t g = cgid ? cgid[(size_t)r * W + e] : (uint32_t)e;
      if ((int64_t)g >= offset && (int64_t)g < offset + Vr) {
        const int c = (int)((int64_t)g - offset);
        atomicOr(&bm[c >> 5], 1u << (c & 31));
        ++kept;
      }
    }
    __syncthreads();
    if (bg_done) {
      // the shard call already wrote the local top-k over a -inf background: only the local
      // candidates that did not survive globally are cleared
      const int nl = kc_s[r];
      for (int i = tid; i < nl; i += kT) {
        const int c = kidx_s[(size_t)r * kmax + i];
        if (!((bm[c >> 5] >> (c & 31)) & 1u)) o[c] = ninf;
      }
    } else {
      for (int c = tid; c < Vr; c += kT) o[c] = (bm[c >> 5] >> (c & 31)) & 1u ? in[c] : ninf;
    }
  } else if (R.mode == MODE_TOPP && R.state == FOUND) {
    uint32_t before = 0u;
    for (int g = 0; g < rank; ++g) before += qbuf[(size_t)r * world + g];
    const uint32_t quota = R.jstar > before ? min(R.jstar - before, R.c_local) : 0u;
    uint32_t run = 0u;
    for (int base = 0; base < Vr; base += kT) {
      const int c = base + tid;
      const uint32_t u = c < Vr ? key_at(in, c) >> sh : 0u;   // compared in the search's key units
      const bool eq = c < Vr && u == R.hi;
      uint32_t tot;
      const uint32_t ord = run + cta_exscan(eq ? 1u : 0u, buf, tot);
      if (c < Vr) {
        const bool keep = u > R.hi || (eq && ord < quota);
        kept += keep ? 1u : 0u;
        o[c] = keep ? in[c] : ninf;
      }
      run += tot;
    }
  } else {  // pass-through rows, keep-all top-p rows (and invalid rows: undefined, copied)
    for (int c = tid; c < Vr; c += kT) {
      if (o != in) o[c] = in[c];
    }
    kept = tid == 0 ? (uint32_t)Vr : 0u;
  }
  if (kept) atomicAdd(&nkept, kept);
  __syncthreads();
  if (tid == 0 && kept_count) kept_count[r] = (int32_t)nkept;
}

// Candidate rows up to kSmallW entries (world * kmax) are resolved in shared memory from sorted
// per-rank lists (tp_pack_sorted + tp_merge_resolve); wider ones by the single-GPU kernels.
constexpr int kSmallW = 16384;

// Descending bitonic sort of NT * EPT composites: blocked in registers (element t * EPT + j in
// thread t), strides < EPT in registers, < 32 * EPT through warp shuffles, larger through `sk`.
template <int NT, int EPT>
__device__ __forceinline__ void bitonic_desc(unsigned long long *sk) {
  constexpr int N = NT * EPT;
  const int tid = threadIdx.x;
  unsigned long long v[EPT];
#pragma unroll
  for (int j = 0; j < EPT; ++j) v[j] = sk[tid * EPT + j];
  for (int size = 2; size <= N; size <<= 1) {
    int stride = size >> 1;
    if (stride >= 32 * EPT) {
#pragma unroll
      for (int j = 0; j < EPT; ++j) sk[tid * EPT + j] = v[j];
      __syncthreads();
      for (; stride >= 32 * EPT; stride >>= 1) {
        for (int t = tid; t < N / 2; t += NT) {
          const int i = ((t & ~(stride - 1)) << 1) | (t & (stride - 1)), j = i | stride;
          const unsigned long long a = sk[i], b = sk[j];
          const bool desc = (i & size) == 0;
          if (desc ? a < b : a > b) { sk[i] = b; sk[j] = a; }
        }
        __syncthreads();
      }
#pragma unroll
      for (int j = 0; j < EPT; ++j) v[j] = sk[tid * EPT + j];
    }
    for (; stride >= EPT; stride >>= 1) {
      const int lm = stride / EPT;
#pragma unroll
      for (int j = 0; j < EPT; ++j) {
        const int i = tid * EPT + j;
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, v[j], lm);
        const bool hi = ((i & stride) == 0) == ((i & size) == 0);
        v[j] = hi ? (v[j] > o ? v[j] : o) : (v[j] < o ? v[j] : o);
      }
    }
#pragma unroll
    for (int s = EPT >> 1; s > 0; s >>= 1) {
      if (s < size) {
#pragma unroll
        for (int j = 0; j < EPT; ++j) {
          if ((j & s) == 0) {
            const bool desc = ((tid * EPT + j) & size) == 0;
            const unsigned long long a = v[j], b = v[j | s];
            if (desc ? a < b : a > b) { v[j] = b; v[j | s] = a; }
          }
        }
      }
    }
  }
  __syncthreads();  // the last shared-memory phase's readers are done
#pragma unroll
  for (int j = 0; j < EPT; ++j) sk[tid * EPT + j] = v[j];
  __syncthreads();
}

// The rank's candidates of row blockIdx.x sorted by (value desc, global column asc): 64-bit
// (order key, ~global column) composites, bitonic in registers / shuffles / shared memory (NT * EPT
// slots >= kmax), so the gathered lists only need merging.  send = [counts | keys | columns].
template <typename T, int NT, int EPT>
__global__ void __launch_bounds__(NT) tp_pack_sorted(const T *logits, int64_t ld, int64_t offset, int kmax,
                                                    const int32_t *kc, const int32_t *kidx, uint32_t *send, int B4,
                                                    int B) {
  extern __shared__ unsigned long long sk[];  // [NT * EPT]
  constexpr int Kp = NT * EPT;
  const int r = blockIdx.x, tid = threadIdx.x;
  const int cnt = kc[r];
  const T *row = logits + (size_t)r * ld;
  for (int i = tid; i < Kp; i += NT) {
    unsigned long long c = 0ull;  // pads sort after every real entry
    if (i < cnt) {
      const int col = kidx[(size_t)r * kmax + i];
      c = ((unsigned long long)key_at(row, col) << 32) | (0xffffffffu - (uint32_t)(offset + col));
    }
    sk[i] = c;
  }
  __syncthreads();
  // the shard call's bin-sort resolve usually emits its kept columns already in this order: sort
  // only when some neighbour pair is out of order
  int unsorted = 0;
  for (int i = tid; i + 1 < cnt; i += NT) unsorted |= sk[i] < sk[i + 1] ? 1 : 0;
  if (__syncthreads_or(unsorted)) bitonic_desc<NT, EPT>(sk);
  uint32_t *keys = send + B4 + (size_t)r * kmax;
  uint32_t *gid = send + B4 + (size_t)B * kmax + (size_t)r * kmax;
  for (int i = tid; i < kmax; i += NT) {
    const unsigned long long c = i < cnt ? sk[i] : 0ull;
    keys[i] = i < cnt ? (uint32_t)(c >> 32) : 0u;
    gid[i] = i < cnt ? 0xffffffffu - (uint32_t)c : 0xffffffffu;
  }
  if (tid == 0) send[r] = (uint32_t)cnt;
}

constexpr int kMergeT = 512;

// The exact answer on one candidate row from the ranks' sorted lists: the global rank of a list's
// i-th entry is i plus, per other list, the count of its entries above it (binary search); the
// entries ranked below k land in rank order (the global top-k, sorted), then — p < 1 — the
// survivors' exact fixed-point normaliser and prefix masses (oracle.py:70-89): the first prefix
// whose exactly rounded sum reaches p, all of them when fsum(survivors) <= p.  Writes the kept
// global columns (kidx_c) and their count (kc_c).
__global__ void __launch_bounds__(kMergeT) tp_merge_resolve(const uint32_t *recv, size_t send_words, int B4, int B,
                                                           int kmax, int world, int scap, int lp, int wp,
                                                           const int64_t *kk, const double *pp, TpRow *rows,
                                                           int32_t *kidx_c, int32_t *kc_c, int W,
                                                           unsigned long long *bnd) {
  // lp: list slots (power of two >= kmax); wp: lists (power of two >= world); lp == 0: no merge tree
  extern __shared__ unsigned long long sk[];  // rank path: [W] lists | [scap] sorted | offsets
  unsigned long long *srt = world > 1 ? sk + W : sk;
  uint32_t *off = reinterpret_cast<uint32_t *>(sk + W + (world > 1 ? scap : 0));  // [world + 1]
  __shared__ uint32_t s_off[kMaxWorld + 1];
  __shared__ Fx scan_buf[kWarps];
  __shared__ uint32_t s_L, s_keep;
  const int r = blockIdx.x, tid = threadIdx.x;
  const int mode = rows[r].mode;
  if (mode != MODE_TOPK && mode != MODE_TOPKP) {
    // top-p-only rows: each shard sent one candidate, its max (tp_merge's rule)
    if (mode == MODE_TOPP && tid == 0) {
      uint32_t mk = 0u;
      for (int g = 0; g < world; ++g) {
        const uint32_t *sg = recv + (size_t)g * send_words;
        if (sg[r]) mk = max(mk, sg[B4 + (size_t)r * kmax]);
      }
      rows[r].maxkey = mk;
    }
    return;
  }
  if (tid == 0) {
    uint32_t acc = 0u;
    for (int g = 0; g < world; ++g) {
      s_off[g] = acc;
      acc += recv[(size_t)g * send_words + r];
    }
    s_off[world] = acc;
  }
  __syncthreads();
  const uint32_t n = s_off[world];
  const int k = (int)min((int64_t)n, kk[r]);
  if (world > 1 && lp > 0 && k <= lp) {
    // merge tree: list g in slots [g * lp, (g + 1) * lp), padded with 0 (below every entry); each
    // level merges list pairs into the top lp of the two (half-cleaner against the reversed partner,
    // then a bitonic merge) until list 0 holds the global top lp in order
    const int lg = 31 - __clz(lp);  // lp = 1 << lg
    for (int e = tid; e < wp * lp; e += kMergeT) {
      const int g = e >> lg, i = e & (lp - 1);
      unsigned long long c = 0ull;
      if (g < world && (uint32_t)i < s_off[g + 1] - s_off[g]) {
        const uint32_t *sg = recv + (size_t)g * send_words;
        c = ((unsigned long long)sg[B4 + (size_t)r * kmax + i] << 32) |
            (0xffffffffu - sg[B4 + (size_t)B * kmax + (size_t)r * kmax + i]);
      }
      sk[e] = c;
    }
    __syncthreads();
    for (int half = 1; half < wp; half <<= 1) {
      const int pairs = wp / (2 * half);
      for (int e = tid; e < pairs * lp; e += kMergeT) {
        const int j = e >> lg, i = e & (lp - 1);
        unsigned long long *A = sk + (size_t)(2 * j * half) * lp, *Bl = sk + (size_t)(2 * j * half + half) * lp;
        const unsigned long long a = A[i], b = Bl[lp - 1 - i];
        A[i] = a > b ? a : b;
      }
      __syncthreads();
      for (int stride = lp >> 1; stride > 0; stride >>= 1) {
        for (int e = tid; e < pairs * (lp >> 1); e += kMergeT) {
          const int j = e >> (lg - 1), t = e & ((lp >> 1) - 1);
          unsigned long long *A = sk + (size_t)(2 * j * half) * lp;
          const int i = ((t & ~(stride - 1)) << 1) | (t & (stride - 1));
          const unsigned long long x = A[i], y = A[i + stride];
          if (x < y) { A[i] = y; A[i + stride] = x; }
        }
        __syncthreads();
      }
    }
    srt = sk;  // list 0: the global top lp >= k, descending
  } else {
  if (tid == 0)
    for (int g = 0; g <= world; ++g) off[g] = s_off[g];
  __syncthreads();
  for (int g = 0; g < world; ++g) {
    const uint32_t *sg = recv + (size_t)g * send_words;
    const uint32_t o = off[g], ng = off[g + 1] - o;
    const uint32_t *keys = sg + B4 + (size_t)r * kmax;
    const uint32_t *gid = sg + B4 + (size_t)B * kmax + (size_t)r * kmax;
    for (uint32_t i = tid; i < ng; i += kMergeT) sk[o + i] = ((unsigned long long)keys[i] << 32) | (0xffffffffu - gid[i]);
  }
  __syncthreads();
  if (world > 1) {
    for (uint32_t e = tid; e < n; e += kMergeT) {
      int lo = 0, hi = world;  // list of e: off[g] <= e < off[g + 1]
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (off[mid] <= e) lo = mid; else hi = mid;
      }
      const int g = lo;
      uint32_t rank = e - off[g];
      if (rank >= (uint32_t)k) continue;
      const unsigned long long c = sk[e];
      for (int h = 0; h < world && rank < (uint32_t)k; ++h) {
        if (h == g) continue;
        uint32_t a = off[h], z = off[h + 1];  // entries of list h above c: a prefix (descending)
        while (a < z) {
          const uint32_t mid = (a + z) >> 1;
          if (sk[mid] > c) a = mid + 1; else z = mid;
        }
        rank += a - off[h];
      }
      if (rank < (uint32_t)k) srt[rank] = c;
    }
    __syncthreads();
  }
  }
  const double p = pp[r];
  if (tid == 0) s_keep = (uint32_t)k;
  if (p < 1.0 && tid < kThreads) {
    const double m = value_of_key((uint32_t)(srt[0] >> 32));
    const int E = (k + kThreads - 1) / kThreads, q0 = tid * E;
    Fx d = fx_zero();
    for (int j = 0; j < E; ++j)
      if (q0 + j < k) d = fx_add(d, fx_from_double(exp(value_of_key((uint32_t)(srt[q0 + j] >> 32)) - m)));
    Fx D_fx;
    (void)block_exscan_fx(d, scan_buf, D_fx);
    const double D = fx_to_double(D_fx);
    Fx ms = fx_zero();
    for (int j = 0; j < E; ++j)
      if (q0 + j < k) ms = fx_add(ms, fx_from_double(exp(value_of_key((uint32_t)(srt[q0 + j] >> 32)) - m) / D));
    tsync();  // scan_buf reuse
    Fx total;
    Fx pre = block_exscan_fx(ms, scan_buf, total);
    if (tid == 0) s_L = (uint32_t)k;
    tsync();
    const Fx Tp = fx_round_threshold(p);
    for (int j = 0; j < E; ++j) {
      if (q0 + j < k) {
        pre = fx_add(pre, fx_from_double(exp(value_of_key((uint32_t)(srt[q0 + j] >> 32)) - m) / D));
        if (fx_ge(pre, Tp)) { atomicMin(&s_L, (uint32_t)(q0 + j + 1)); break; }
      }
    }
    tsync();
    if (tid == 0 && fx_ge(total, fx_round_threshold(nextafter(p, 2.0)))) s_keep = s_L;  // oracle.py:44-46
  }
  __syncthreads();
  const int L = (int)s_keep;
  for (int i = tid; i < L; i += kMergeT) kidx_c[(size_t)r * W + i] = (int32_t)(0xffffffffu - (uint32_t)srt[i]);
  if (tid == 0) {
    kc_c[r] = L;
    bnd[r] = L > 0 ? srt[L - 1] : ~0ull;  // the kept set is every candidate at or above this composite
  }
}

// ------------------------------------------------------------------------------------------------
// workspace layout
// ------------------------------------------------------------------------------------------------
struct TpLayout {
  int kmax, W, B4;
  size_t send_words;
  size_t ws0, ws0_bytes, ws1, ws1_bytes, k_loc, p_one, k_c, p_c, kc_s, kidx_s, send, recv, cval, cgid, kidx_c,
      kc_c, bnd, rows, tst, dl, part, part_loc, qbuf, total;
};

inline TpLayout tp_layout(int B, int Vr, int world, int k_cap) {
  TpLayout L;
  L.kmax = k_cap < 1 ? 1 : k_cap;
  if (L.kmax > Vr) L.kmax = Vr;
  L.kmax = (L.kmax + 3) & ~3;  // 16-byte candidate rows: the resolve runs on the fused kernel
  L.W = world * L.kmax;
  L.B4 = (B + 3) & ~3;
  L.send_words = (size_t)L.B4 + 2ull * (size_t)B * (size_t)L.kmax;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  L.ws0_bytes = align_up(ws_layout(B, Vr).total, 256);
  L.ws0 = take(L.ws0_bytes);  // the shard call's workspace first: its status block is the call's
  L.ws1_bytes = align_up(ws_layout(B, L.W).total, 256);
  L.ws1 = take(L.ws1_bytes);
  L.k_loc = take(8ull * B);
  L.p_one = take(8ull * B);
  L.k_c = take(8ull * B);
  L.p_c = take(8ull * B);
  L.kc_s = take(4ull * B);
  L.kidx_s = take(4ull * B * L.kmax);
  L.send = take(4ull * L.send_words);
  L.recv = take(4ull * L.send_words * (size_t)world);
  L.cval = take(4ull * B * L.W);
  L.cgid = take(4ull * B * L.W);
  L.kidx_c = take(4ull * B * L.W);
  L.kc_c = take(4ull * B);
  L.bnd = take(8ull * B);
  L.rows = take(sizeof(TpRow) * (size_t)B);
  L.tst = take(4ull * B);
  L.dl = take(8ull * 4 * B);
  L.part = take(8ull * kPartWords * B);
  L.part_loc = take(8ull * kPartWords * B);
  L.qbuf = take(4ull * B * (size_t)world);
  L.total = off;
  return L;
}

// ------------------------------------------------------------------------------------------------
// NCCL, loaded at run time (libnccl.so.2 is usually already in the process through torch)
// ------------------------------------------------------------------------------------------------
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId *);
  ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int);
  ncclResult_t (*comm_destroy)(ncclComm_t);
  ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*all_gather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
};

const NcclApi *nccl_api() {
  static NcclApi api;
  static bool ok = false;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
    api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
    api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
    api.all_reduce = (decltype(api.all_reduce))dlsym(h, "ncclAllReduce");
    api.all_gather = (decltype(api.all_gather))dlsym(h, "ncclAllGather");
    ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce && api.all_gather;
  });
  return ok ? &api : nullptr;
}

int nccl_all_reduce_sum(void *buf, size_t count, int elem_bytes, qrita_stream_t st, void *ctx) {
  const NcclApi *a = nccl_api();
  if (!a) return 1;
  return a->all_reduce(buf, buf, count, elem_bytes == 8 ? ncclUint64 : ncclUint32, ncclSum, (ncclComm_t)ctx,
                       (cudaStream_t)st) == ncclSuccess ? 0 : 1;
}

int nccl_all_gather(const void *send, void *recv, size_t bytes, qrita_stream_t st, void *ctx) {
  const NcclApi *a = nccl_api();
  if (!a) return 1;
  return a->all_gather(send, recv, bytes, ncclUint8, (ncclComm_t)ctx, (cudaStream_t)st) == ncclSuccess ? 0 : 1;
}

template <typename K>
cudaError_t smem_optin(K kernel, int *slots) {
  int v = 0;
  return per_device_once(slots, [&](int, int &out) {
    out = 1;
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(210u << 10));
  }, v);
}

template <typename T, int NT, int EPT>
cudaError_t launch_pack(const T *x, int64_t ld, int64_t offset, const TpLayout &L, const int32_t *kc,
                        const int32_t *kidx, uint32_t *send, int B, cudaStream_t st) {
  constexpr size_t sbytes = (size_t)NT * EPT * 8;
  static int optin[kMaxDevices] = {};
  if (sbytes > (48u << 10) && smem_optin(tp_pack_sorted<T, NT, EPT>, optin) != cudaSuccess) return cudaErrorUnknown;
  tp_pack_sorted<T, NT, EPT><<<B, NT, sbytes, st>>>(x, ld, offset, L.kmax, kc, kidx, send, L.B4, B);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_pack_sorted(const T *x, int64_t ld, int64_t offset, const TpLayout &L, const int32_t *kc,
                               const int32_t *kidx, uint32_t *send, int B, cudaStream_t st) {
  const int km = L.kmax;
  if (km <= 256) return launch_pack<T, 256, 1>(x, ld, offset, L, kc, kidx, send, B, st);
  if (km <= 512) return launch_pack<T, 256, 2>(x, ld, offset, L, kc, kidx, send, B, st);
  if (km <= 1024) return launch_pack<T, 256, 4>(x, ld, offset, L, kc, kidx, send, B, st);
  if (km <= 2048) return launch_pack<T, 256, 8>(x, ld, offset, L, kc, kidx, send, B, st);
  if (km <= 4096) return launch_pack<T, 256, 16>(x, ld, offset, L, kc, kidx, send, B, st);
  if (km <= 8192) return launch_pack<T, 512, 16>(x, ld, offset, L, kc, kidx, send, B, st);
  return launch_pack<T, 1024, 16>(x, ld, offset, L, kc, kidx, send, B, st);
}

// tp_merge_resolve's merge tree: list slots (power of two >= kmax) and lists (power of two >= world)
inline void merge_tree_shape(const TpLayout &L, int world, int &lp, int &wp) {
  lp = 1;
  while (lp < L.kmax) lp <<= 1;
  wp = 1;
  while (wp < world) wp <<= 1;
  if (world < 2 || (size_t)lp * wp * 8 > (200u << 10)) lp = 0;  // rank path only
}

// shared memory of tp_merge_resolve: the rank path's lists + sorted top-k + offsets, or the tree
inline size_t merge_smem(const TpLayout &L, int world, int scap) {
  int lp, wp;
  merge_tree_shape(L, world, lp, wp);
  const size_t rank_path = (size_t)L.W * 8 + (world > 1 ? (size_t)scap * 8 : 0) + (size_t)(world + 1) * 4;
  const size_t tree = (size_t)lp * wp * 8;
  return rank_path > tree ? rank_path : tree;
}

template <typename T>
int run_tp(const void *logits, int64_t ld_in, int dtype, int B, int Vr, int Vg, int64_t offset, const int64_t *k,
           const double *p, int k_cap, void *out, int64_t ld_out, int32_t *kept_count, void *workspace,
           size_t ws_bytes, int flags, int rank, int world, const qrita_comm *comm, cudaStream_t st) {
  const TpLayout L = tp_layout(B, Vr, world, k_cap);
  if (ws_bytes < L.total || ((uintptr_t)workspace & 255u)) return QRITA_EWORKSPACE;
  uint8_t *ws = (uint8_t *)workspace;
  auto at = [&](size_t o) { return (void *)(ws + o); };
  const int sh = dtype == QRITA_DTYPE_BF16 ? 16 : 0;
  const int npass = dtype == QRITA_DTYPE_BF16 ? 4 : 8;
  const size_t bm_bytes = (size_t)((Vr + 31) / 32) * 4;
  static int optin_pack[kMaxDevices] = {}, optin_write[kMaxDevices] = {};
  if (bm_bytes > (48u << 10)) {
    if (smem_optin(tp_pack<T>, optin_pack) != cudaSuccess || smem_optin(tp_write<T>, optin_write) != cudaSuccess)
      return QRITA_ECUDA;
  }
  const T *x = (const T *)logits;
  const int scap = L.W < ((k_cap + 3) & ~3) ? L.W : ((k_cap + 3) & ~3);  // sorted top-k slots
  // candidate rows resolved in shared memory (tp_pack_sorted + tp_merge_resolve)
  const bool small = L.W <= kSmallW && merge_smem(L, world, scap) <= (210u << 10);
  int64_t *k_loc = (int64_t *)at(L.k_loc), *k_c = (int64_t *)at(L.k_c);
  double *p_one = (double *)at(L.p_one), *p_c = (double *)at(L.p_c);
  TpRow *rows = (TpRow *)at(L.rows);
  int32_t *tst = (int32_t *)at(L.tst);
  const bool no_topp = (flags & QRITA_TP_NO_TOPP_ROWS) != 0;
  tp_prep<<<(B + 255) / 256, 256, 0, st>>>(B, Vg, Vr, k_cap < 1 ? 1 : k_cap, no_topp ? 1 : 0, k, p, k_loc, p_one,
                                          rows, tst);
  if (cudaGetLastError() != cudaSuccess) return QRITA_ECUDA;
  // (1) local top-k_loc of the shard: its kept columns, and — when no row needs the whole shard
  //     (no top-p-only rows) and the output is a separate buffer — the local top-k over a -inf
  //     background straight into `out` (the final write then only clears dropped candidates)
  const bool bg = no_topp && out != logits;
  int rc = topk_topp_impl(logits, ld_in, dtype, B, Vr, k_loc, p_one, bg ? out : nullptr, bg ? ld_out : Vr,
                          (int32_t *)at(L.kc_s), nullptr, at(L.ws0), L.ws0_bytes, 0, 4096, (qrita_stream_t)st,
                          nullptr, nullptr, nullptr, nullptr, (int32_t *)at(L.kidx_s), L.kmax);
  if (rc != QRITA_OK) return rc;
  if (small) {
    if (launch_pack_sorted<T>(x, ld_in, offset, L, (const int32_t *)at(L.kc_s), (const int32_t *)at(L.kidx_s),
                              (uint32_t *)at(L.send), B, st) != cudaSuccess)
      return QRITA_ECUDA;
  } else {
    tp_pack<T><<<B, kT, bm_bytes, st>>>(x, ld_in, Vr, offset, L.kmax, (const int32_t *)at(L.kc_s),
                                        (const int32_t *)at(L.kidx_s), (uint32_t *)at(L.send), L.B4, B, 1);
    if (cudaGetLastError() != cudaSuccess) return QRITA_ECUDA;
  }
  if (comm->all_gather(at(L.send), at(L.recv), 4 * L.send_words, (qrita_stream_t)st, comm->ctx) != 0)
    return QRITA_ENCCL;
  // (2) the exact answer on the gathered candidates (same on every rank): a shared-memory sort for
  //     candidate rows up to kSmallW entries, else the single-GPU kernels
  if (small) {
    const size_t sb = merge_smem(L, world, scap);
    static int optin_merge[kMaxDevices] = {};
    if (sb > (48u << 10) && smem_optin(tp_merge_resolve, optin_merge) != cudaSuccess) return QRITA_ECUDA;
    int lp, wp;
    merge_tree_shape(L, world, lp, wp);
    tp_merge_resolve<<<B, kMergeT, sb, st>>>((const uint32_t *)at(L.recv), L.send_words, L.B4, B, L.kmax, world,
                                             scap, lp, wp, k, p, rows, (int32_t *)at(L.kidx_c), (int32_t *)at(L.kc_c),
                                             L.W, (unsigned long long *)at(L.bnd));
    if (cudaGetLastError() != cudaSuccess) return QRITA_ECUDA;
  } else {
    tp_merge<<<B, kT, 0, st>>>((const uint32_t *)at(L.recv), L.send_words, L.B4, B, L.kmax, world, L.W, k, p, rows,
                               (float *)at(L.cval), (uint32_t *)at(L.cgid), k_c, p_c);
    if (cudaGetLastError() != cudaSuccess) return QRITA_ECUDA;
    rc = topk_topp_impl(at(L.cval), L.W, QRITA_DTYPE_F32, B, L.W, k_c, p_c, nullptr, L.W, (int32_t *)at(L.kc_c),
                        nullptr, at(L.ws1), L.ws1_bytes, 0, 4096, (qrita_stream_t)st, nullptr, nullptr, nullptr,
                        nullptr, (int32_t *)at(L.kidx_c), L.W);
    if (rc != QRITA_OK) return rc;
  }
  // (3) top-p-only rows: exact normaliser, radix boundary search, tie quotas
  if (!no_topp) {
    unsigned long long *dl = (unsigned long long *)at(L.dl), *part = (unsigned long long *)at(L.part),
                       *part_loc = (unsigned long long *)at(L.part_loc);
    tp_denom<T><<<B, kT, 0, st>>>(x, ld_in, Vr, p, rows, dl, sh);
    if (cudaGetLastError() != cudaSuccess) return QRITA_ECUDA;
    if (comm->all_reduce_sum(dl, 4ull * B, 8, (qrita_stream_t)st, comm->ctx) != 0) return QRITA_ENCCL;
    for (int q = 0; q < npass; ++q) {
      tp_pass<T><<<B, kT, 0, st>>>(x, ld_in, Vr, rows, dl, part, part_loc, q, sh);
      if (cudaGetLastError() != cudaSuccess) return QRITA_ECUDA;
      if (comm->all_reduce_sum(part, (size_t)kPartWords * B, 8, (qrita_stream_t)st, comm->ctx) != 0)
        return QRITA_ENCCL;
    }
    tp_quota<<<(B + 127) / 128, 128, 0, st>>>(B, rows, part, part_loc, (uint32_t *)at(L.qbuf), rank, world, sh);
    if (cudaGetLastError() != cudaSuccess) return QRITA_ECUDA;
    if (comm->all_reduce_sum(at(L.qbuf), (size_t)B * world, 4, (qrita_stream_t)st, comm->ctx) != 0)
      return QRITA_ENCCL;
  }
  // (4) the shard output
  const WsLayout W0 = ws_layout(B, Vr);
  tp_write<T><<<B, kT, (small && bg) ? 0 : bm_bytes, st>>>(x, ld_in, (T *)out, ld_out, Vr, offset, rows,
                                       small ? nullptr : (const uint32_t *)at(L.cgid),
                                       (const int32_t *)at(L.kidx_c), (const int32_t *)at(L.kc_c), L.W,
                                       (const uint32_t *)at(L.qbuf), rank, world, kept_count,
                                       (int32_t *)(ws + L.ws0 + W0.status), tst, sh, bg ? 1 : 0,
                                       (const int32_t *)at(L.kidx_s), (const int32_t *)at(L.kc_s), L.kmax,
                                       small ? (const unsigned long long *)at(L.bnd) : nullptr,
                                       (const uint32_t *)at(L.send), L.B4, B);
  return cudaGetLastError() == cudaSuccess ? QRITA_OK : QRITA_ECUDA;
}

}  // namespace tp
}  // namespace qrita

using namespace qrita;

extern "C" {

size_t qrita_tp_workspace_bytes(int B, int V_shard, int dtype, int world, int k_cap) {
  (void)dtype;
  if (B < 1 || V_shard < 1 || world < 1) return 0;
  return tp::tp_layout(B, V_shard, world, k_cap).total;
}

int qrita_topk_topp_tp_comm(const void *logits, int64_t ld_in, int dtype, int B, int V_shard, int V_global,
                            int64_t vocab_offset, const int64_t *k, const double *p, int k_cap, void *out,
                            int64_t ld_out, int32_t *kept_count, void *workspace, size_t ws_bytes, int flags,
                            int rank, int world, const qrita_comm *comm, qrita_stream_t stream) {
  if (!logits || !out || !k || !p || !workspace || !comm || !comm->all_reduce_sum || !comm->all_gather)
    return QRITA_EINVAL_ARG;
  if (B < 1 || V_shard < 1 || V_shard > tp::kMaxShard || V_global < V_shard || ld_in < V_shard ||
      ld_out < V_shard || world < 1 || world > tp::kMaxWorld || rank < 0 || rank >= world || vocab_offset < 0 ||
      vocab_offset + V_shard > (int64_t)V_global)
    return QRITA_EINVAL_ARG;
  if (dtype != QRITA_DTYPE_F32 && dtype != QRITA_DTYPE_BF16) return QRITA_EINVAL_ARG;
  if (flags & ~(QRITA_INPLACE | QRITA_TP_NO_TOPP_ROWS)) return QRITA_EINVAL_ARG;
  if (((flags & QRITA_INPLACE) != 0) != (logits == out)) return QRITA_EINVAL_ARG;
  if (dtype == QRITA_DTYPE_F32)
    return tp::run_tp<float>(logits, ld_in, dtype, B, V_shard, V_global, vocab_offset, k, p, k_cap, out, ld_out,
                             kept_count, workspace, ws_bytes, flags, rank, world, comm, (cudaStream_t)stream);
  return tp::run_tp<uint16_t>(logits, ld_in, dtype, B, V_shard, V_global, vocab_offset, k, p, k_cap, out, ld_out,
                              kept_count, workspace, ws_bytes, flags, rank, world, comm, (cudaStream_t)stream);
}

int qrita_topk_topp_tp(const void *logits, int64_t ld_in, int dtype, int B, int V_shard, int V_global,
                       int64_t vocab_offset, const int64_t *k, const double *p, int k_cap, void *out, int64_t ld_out,
                       int32_t *kept_count, void *workspace, size_t ws_bytes, int flags, int rank, int world,
                       void *nccl_comm, qrita_stream_t stream) {
  if (!nccl_comm) return QRITA_EINVAL_ARG;
  if (!tp::nccl_api()) return QRITA_ENCCL;
  qrita_comm c{tp::nccl_all_reduce_sum, tp::nccl_all_gather, nccl_comm};
  return qrita_topk_topp_tp_comm(logits, ld_in, dtype, B, V_shard, V_global, vocab_offset, k, p, k_cap, out, ld_out,
                                 kept_count, workspace, ws_bytes, flags, rank, world, &c, stream);
}

int qrita_nccl_unique_id(void *id_out) {
  const tp::NcclApi *a = tp::nccl_api();
  if (!a || !id_out) return QRITA_ENCCL;
  ncclUniqueId id;
  if (a->get_unique_id(&id) != ncclSuccess) return QRITA_ENCCL;
  memcpy(id_out, &id, sizeof(id));
  return QRITA_OK;
}

int qrita_nccl_comm_init(void **comm_out, int world, const void *id, int rank) {
  const tp::NcclApi *a = tp::nccl_api();
  if (!a || !comm_out || !id) return QRITA_ENCCL;
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  if (a->comm_init_rank(&c, world, uid, rank) != ncclSuccess) return QRITA_ENCCL;
  *comm_out = (void *)c;
  return QRITA_OK;
}

int qrita_nccl_comm_destroy(void *comm) {
  const tp::NcclApi *a = tp::nccl_api();
  if (!a || !comm) return QRITA_ENCCL;
  return a->comm_destroy((ncclComm_t)comm) == ncclSuccess ? QRITA_OK : QRITA_ENCCL;
}

int qrita_copy_sync(void *dst, const void *src, size_t bytes, qrita_stream_t stream) {
  if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream) != cudaSuccess) return QRITA_ECUDA;
  return cudaStreamSynchronize((cudaStream_t)stream) == cudaSuccess ? QRITA_OK : QRITA_ECUDA;
}

}  // extern "C"
