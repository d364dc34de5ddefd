// Microbenchmark: direct-mapped 16-bit shared-memory histograms of bf16 order keys (cfg3-like rows),
// C CTAs per row, T threads per CTA; plain atomics vs match_any warp aggregation.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t key16(uint16_t b) {
  uint32_t x = ((uint32_t)b) << 16;
  if ((x << 1) == 0u) x = 0u;
  x = (x & 0x80000000u) ? ~x : (x | 0x80000000u);
  return x >> 16;
}

template <int AGG>
__global__ void hist_kernel(const uint16_t *x, int V, int C, uint32_t *sink) {
  extern __shared__ uint32_t h[];
  const int row = blockIdx.x / C, q = blockIdx.x % C;
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) h[i] = 0u;
  __syncthreads();
  const int L = (V + C - 1) / C;
  const int lo = q * L, hi = min(V, lo + L);
  const uint16_t *r = x + (size_t)row * V;
  for (int c = lo + threadIdx.x * 8; c < hi; c += blockDim.x * 8) {
    uint4 v = *reinterpret_cast<const uint4 *>(r + c);
    uint16_t e[8];
    memcpy(e, &v, 16);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t u = key16(e[j]);
      if (AGG) {
        const unsigned peers = __match_any_sync(0xffffffffu, u);
        const int leader = __ffs(peers) - 1;
        if ((threadIdx.x & 31) == leader) atomicAdd(&h[u >> 1], (uint32_t)__popc(peers) << ((u & 1) * 16));
      } else {
        atomicAdd(&h[u >> 1], 1u << ((u & 1) * 16));
      }
    }
  }
  __syncthreads();
  uint32_t s = 0;
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) s += h[i];
  if (s == 0xdeadbeef) sink[0] = s;
}

int main() {
  const int B = 64, V = 151936;
  std::vector<uint16_t> hx((size_t)B * V);
  uint64_t st = 12345;
  auto rnd = [&]() { st = st * 6364136223846793005ull + 1442695040888963407ull; return (double)(st >> 11) / 9007199254740992.0; };
  for (size_t i = 0; i < hx.size(); i += 2) {
    double u1 = rnd() + 1e-300, u2 = rnd();
    double r = sqrt(-2 * log(u1));
    double z[2] = {r * cos(6.283185307179586 * u2), r * sin(6.283185307179586 * u2)};
    for (int j = 0; j < 2; ++j) {
      float f = (float)z[j];
      if (f < 0) f = roundf(4 * f) / 4;
      uint32_t b;
      memcpy(&b, &f, 4);
      hx[i + j] = (uint16_t)((b + 0x7fff + ((b >> 16) & 1)) >> 16);
    }
  }
  uint16_t *dx;
  uint32_t *sink;
  cudaMalloc(&dx, hx.size() * 2);
  cudaMalloc(&sink, 4);
  cudaMemcpy(dx, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(hist_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(hist_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int agg = 0; agg < 2; ++agg)
    for (int C : {1, 2, 4})
      for (int T : {256, 512, 1024}) {
        float best = 1e9;
        for (int it = 0; it < 5; ++it) {
          cudaEventRecord(a);
          if (agg) hist_kernel<1><<<B * C, T, 131072>>>(dx, V, C, sink);
          else hist_kernel<0><<<B * C, T, 131072>>>(dx, V, C, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (ms < best) best = ms;
        }
        printf("agg=%d C=%d T=%4d: %8.1f us  %s\n", agg, C, T, best * 1e3, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
