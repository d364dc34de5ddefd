// qrita_device.cuh — device building blocks shared by the truncation kernels.
//
//  * order keys: fp32 bit patterns mapped to uint32 so that integer order == the reference's
//    stable-sort value order (oracle.py:16-18 sorts -float64(z); -0.0 and +0.0 compare equal there,
//    so both map to the same key here);
//  * Fx: an exact 192-bit fixed-point accumulator (unit 2^-128) for fp64 probability masses.  Sums
//    are exact and therefore independent of reduction order, which is what makes the nucleus test
//    reproduce math.fsum (oracle.py:37-54, pivot_search.py:143-196) and run-to-run deterministic;
//  * block-wide reductions built on redux.sync (warp) + shared memory (block).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace qrita {

constexpr int kThreads = 256;  // row-tail CTA size
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kNoCut = 0xffffffffu;

// ------------------------------------------------------------------------------------------------
// Order keys
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t canon_bits(uint32_t b) { return (b << 1) == 0u ? 0u : b; }

__device__ __forceinline__ uint32_t key_of_bits(uint32_t b) {
  b = canon_bits(b);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ uint32_t bits_of_key(uint32_t k) {
  return (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
}

__device__ __forceinline__ double value_of_key(uint32_t k) {
  return (double)__uint_as_float(bits_of_key(k));
}

__device__ __forceinline__ bool bits_nonfinite(uint32_t b) {
  return (b & 0x7f800000u) == 0x7f800000u;
}

// ------------------------------------------------------------------------------------------------
// 192-bit unsigned fixed point, value = (w2*2^128 + w1*2^64 + w0) * 2^-128
// ------------------------------------------------------------------------------------------------
struct Fx {
  unsigned long long w0, w1, w2;
};

__device__ __forceinline__ Fx fx_zero() { return Fx{0ull, 0ull, 0ull}; }

__device__ __forceinline__ bool fx_is_zero(const Fx &a) { return (a.w0 | a.w1 | a.w2) == 0ull; }

__device__ __forceinline__ Fx fx_add(const Fx &a, const Fx &b) {
  Fx r;
  asm("add.cc.u64 %0, %3, %6;\n\t"
      "addc.cc.u64 %1, %4, %7;\n\t"
      "addc.u64 %2, %5, %8;"
      : "=l"(r.w0), "=l"(r.w1), "=l"(r.w2)
      : "l"(a.w0), "l"(a.w1), "l"(a.w2), "l"(b.w0), "l"(b.w1), "l"(b.w2));
  return r;
}

// a - b, requires a >= b
__device__ __forceinline__ Fx fx_sub(const Fx &a, const Fx &b) {
  Fx r;
  asm("sub.cc.u64 %0, %3, %6;\n\t"
      "subc.cc.u64 %1, %4, %7;\n\t"
      "subc.u64 %2, %5, %8;"
      : "=l"(r.w0), "=l"(r.w1), "=l"(r.w2)
      : "l"(a.w0), "l"(a.w1), "l"(a.w2), "l"(b.w0), "l"(b.w1), "l"(b.w2));
  return r;
}

// a >= b
__device__ __forceinline__ bool fx_ge(const Fx &a, const Fx &b) {
  if (a.w2 != b.w2) return a.w2 > b.w2;
  if (a.w1 != b.w1) return a.w1 > b.w1;
  return a.w0 >= b.w0;
}

__device__ __forceinline__ Fx fx_add_unit(const Fx &a) { return fx_add(a, Fx{1ull, 0ull, 0ull}); }

// Exact conversion of a non-negative finite double (truncated below 2^-128).
__device__ __forceinline__ Fx fx_from_double(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  int e = (int)((b >> 52) & 0x7ff);
  unsigned long long m = b & ((1ull << 52) - 1ull);
  if (e == 0) {
    if (m == 0ull) return fx_zero();
    e = 1;
  } else {
    m |= 1ull << 52;
  }
  // x = m * 2^(e-1075); fixed = m * 2^(e-947)
  int s = e - 947;
  Fx r = fx_zero();
  if (s < 0) {
    if (s > -64) r.w0 = m >> (-s);
    return r;
  }
  int limb = s >> 6, off = s & 63;
  unsigned long long lo = m << off;
  unsigned long long hi = off ? (m >> (64 - off)) : 0ull;
  if (limb == 0) {
    r.w0 = lo; r.w1 = hi;
  } else if (limb == 1) {
    r.w1 = lo; r.w2 = hi;
  } else if (limb == 2) {
    r.w2 = lo;
  }
  return r;
}

// a * j (j < 2^32), exact while the product stays below 2^64 (integer part).
__device__ __forceinline__ Fx fx_mul_u32(const Fx &a, uint32_t j) {
  unsigned long long jj = j;
  Fx r;
  unsigned long long lo0 = a.w0 * jj, hi0 = __umul64hi(a.w0, jj);
  unsigned long long lo1 = a.w1 * jj, hi1 = __umul64hi(a.w1, jj);
  unsigned long long lo2 = a.w2 * jj;
  r.w0 = lo0;
  r.w1 = lo1 + hi0;
  unsigned long long c = r.w1 < lo1 ? 1ull : 0ull;
  r.w2 = lo2 + hi1 + c;
  return r;
}

// Correctly rounded (nearest-even) conversion to double.  No dynamically indexed arrays (those
// would live in local memory): the top non-zero word is selected explicitly.
__device__ __forceinline__ double fx_to_double(const Fx &a) {
  unsigned long long hi, mid, lo;
  int base;  // bit index of hi's least significant bit in the 192-bit integer
  if (a.w2) { hi = a.w2; mid = a.w1; lo = a.w0; base = 128; }
  else if (a.w1) { hi = a.w1; mid = a.w0; lo = 0ull; base = 64; }
  else {
    // an integer < 2^64: cvt.rn rounds correctly, the power-of-two scale is exact
    return a.w0 ? ldexp(__ull2double_rn(a.w0), -128) : 0.0;
  }
  const int lz = __clzll((long long)hi);
  // 64-bit window starting at the top set bit, plus a sticky bit for everything below it
  const unsigned long long win = lz ? (hi << lz) | (mid >> (64 - lz)) : hi;
  const unsigned long long rest = (lz ? (mid << lz) : mid) | lo;
  return ldexp(__ull2double_rn(rest ? (win | 1ull) : win), base - lz - 128);
}

// Smallest fixed-point value S with round_to_nearest_even(S) >= p, for a double 0 < p <= 1.
// (fsum(prefix) >= p  <=>  exact(prefix) >= fx_round_threshold(p).)
__device__ __forceinline__ Fx fx_round_threshold(double p) {
  if (!(p > 0.0)) return Fx{1ull, 0ull, 0ull};
  if (p < 0x1p-70) {
    // every non-empty prefix already holds >= 1/V >> p; the first positive mass crosses.
    return Fx{1ull, 0ull, 0ull};
  }
  double q = nextafter(p, 0.0);
  Fx P = fx_from_double(p);
  Fx Q = fx_from_double(q);
  Fx s = fx_add(P, Q);
  // halve (exact: both are multiples of >= 2^5 units here)
  Fx mid;
  mid.w0 = (s.w0 >> 1) | (s.w1 << 63);
  mid.w1 = (s.w1 >> 1) | (s.w2 << 63);
  mid.w2 = s.w2 >> 1;
  unsigned long long pb = (unsigned long long)__double_as_longlong(p);
  bool even = (pb & 1ull) == 0ull;
  return even ? mid : fx_add_unit(mid);
}

// ------------------------------------------------------------------------------------------------
// L2 cache policies
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long l2_evict_last_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_keep_u32(uint32_t *p, uint32_t v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" :: "l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep_u4(uint4 *p, uint4 v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol) : "memory");
}

// ------------------------------------------------------------------------------------------------
// Programmatic dependent launch (griddepcontrol, sm_90+)
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// The ring's chunk-sequence words (written by the producing lane, polled by the consuming warps) are
// accessed with atomics only: ordered under the memory model and racecheck-clean (a volatile poll is
// formally a data race).  The distinct-value hash table keeps plain volatile probes on purpose: they
// are independent loads (the batch of probes is in flight together), a stale probe only sends the
// thread to the atomicCAS insert, which decides; racecheck reports those probes.
__device__ __forceinline__ uint32_t ld_relaxed_smem(uint32_t *p) { return atomicOr(p, 0u); }
__device__ __forceinline__ void st_relaxed_smem(uint32_t *p, uint32_t v) { atomicExch(p, v); }

// Barrier of the row-tail thread group (named barrier 1, kThreads threads), in the non-aligned form
// (`barrier.sync`; `bar.sync` is `barrier.sync.aligned`).  Callers reach it right after
// thread-0-only branches and the compiler does not treat inline asm as a barrier, so a warp may
// arrive diverged: undefined behaviour for the aligned form, and a deadlock was observed (even with
// a __syncwarp() in front).  Measured: no cost on the hot path.
__device__ __forceinline__ void tsync() { asm volatile("barrier.sync 1, %0;" :: "n"(kThreads) : "memory"); }

// ------------------------------------------------------------------------------------------------
// mbarrier / bulk-copy (TMA) primitives for the fused kernel's chunk ring
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}"
               :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long *bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.release.cta.shared::cta.b64 st, [%0], %1;\n\t}"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\t"
               "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
               "selp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0u;
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// Bulk global -> shared copy completing on an mbarrier (bytes: multiple of 16, both ends 16-B aligned).
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, unsigned long long *bar,
                                            unsigned long long policy) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy) : "memory");
}
// 16-byte streaming store of one 32-bit word repeated four times (the -inf background: one register).
__device__ __forceinline__ void st_cs_splat4(void *p, uint32_t w) {
  asm volatile("st.global.cs.v4.b32 [%0], {%1, %1, %1, %1};" :: "l"(p), "r"(w) : "memory");
}
// Bulk prefetch of global memory into L2 (no shared memory, no completion tracking).
__device__ __forceinline__ void l2_prefetch_bulk(const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ unsigned long long l2_evict_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// ------------------------------------------------------------------------------------------------
// Warp / block reductions
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t warp_sum(uint32_t v) { return __reduce_add_sync(0xffffffffu, v); }
__device__ __forceinline__ uint32_t warp_min(uint32_t v) { return __reduce_min_sync(0xffffffffu, v); }
__device__ __forceinline__ uint32_t warp_max(uint32_t v) { return __reduce_max_sync(0xffffffffu, v); }

// An Fx split into twelve 16-bit pieces so that warp sums need no carry handling
// (32 lanes * 16 warps * 0xffff < 2^32).
struct FxPieces {
  uint32_t q[12];
};

__device__ __forceinline__ void fx_split(const Fx &a, uint32_t q[12]) {
  const unsigned long long w[3] = {a.w0, a.w1, a.w2};
#pragma unroll
  for (int i = 0; i < 12; ++i) q[i] = (uint32_t)((w[i >> 2] >> ((i & 3) * 16)) & 0xffffull);
}

__device__ __forceinline__ Fx fx_join(const uint32_t q[12]) {
  // q[i] may exceed 16 bits (sums); propagate carries upward.
  unsigned long long w[3] = {0ull, 0ull, 0ull};
  unsigned long long carry = 0ull;
#pragma unroll
  for (int i = 0; i < 12; ++i) {
    unsigned long long v = (unsigned long long)q[i] + carry;
    w[i >> 2] |= (v & 0xffffull) << ((i & 3) * 16);
    carry = v >> 16;
  }
  return Fx{w[0], w[1], w[2]};
}

}  // namespace qrita
