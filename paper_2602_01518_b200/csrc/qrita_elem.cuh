// qrita_elem.cuh — sigma tables, element / vector access, value comparisons.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "qrita_tables.h"
#include "qrita_types.cuh"

namespace qrita {

// The two 200-entry quantile tables (qrita_tables.h).
static __constant__ double c_topk_table[kTableSize] = {QRITA_TOPK_TABLE_VALUES};
static __constant__ double c_topp_table[kTableSize] = {QRITA_TOPP_TABLE_VALUES};

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

// Float helpers of the streaming passes
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

}  // namespace qrita
