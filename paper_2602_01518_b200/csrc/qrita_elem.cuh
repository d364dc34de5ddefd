// qrita_elem.cuh — sigma tables, element / vector access, value comparisons.
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
