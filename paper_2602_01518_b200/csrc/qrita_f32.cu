// fp32 instantiation of the truncation kernels.
#include "qrita_impl.cuh"

namespace qrita {
cudaError_t launch_f32(const Params &P, cudaStream_t st, bool vec, cudaEvent_t prep_done,
                       cudaEvent_t stream_done) {
  return launch_all<float>(P, st, vec, prep_done, stream_done);
}
}  // namespace qrita
