// bf16 instantiation of the truncation kernels (bf16 carried as raw uint16 bits).
#include "qrita_impl.cuh"

namespace qrita {
cudaError_t launch_bf16(const Params &P, cudaStream_t st, bool vec, cudaEvent_t prep_done,
                        cudaEvent_t stream_done) {
  return launch_all<uint16_t>(P, st, vec, prep_done, stream_done);
}
}  // namespace qrita
