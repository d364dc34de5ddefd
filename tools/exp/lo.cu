#include <cuda_runtime.h>
#include <stdint.h>
__global__ void k_empty(int *p) { if (p && threadIdx.x == 9999) *p = 1; }
__global__ void __launch_bounds__(256, 2) k_smem(int *p) {
  extern __shared__ int s[];
  if (p && threadIdx.x == 9999) *p = s[3];
}
// stack-using kernel: local array indexed dynamically
__global__ void __launch_bounds__(256, 2) k_stack(int *p, int n) {
  extern __shared__ int s[];
  int loc[300];
  for (int i = 0; i < 300; ++i) loc[(i * n + threadIdx.x) % 300] = i * n;
  if (p && threadIdx.x == 9999) *p = loc[(n * threadIdx.x) % 300] + s[3];
}
extern "C" int lo_launch(int which, int grid, int smem, void *stream) {
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
    cudaFuncSetAttribute(k_stack, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
    init = true;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (which == 0) k_empty<<<grid, 256, 0, st>>>(nullptr);
  else if (which == 1) k_smem<<<grid, 256, smem, st>>>(nullptr);
  else k_stack<<<grid, 256, smem, st>>>(nullptr, 3);
  return (int)cudaGetLastError();
}
