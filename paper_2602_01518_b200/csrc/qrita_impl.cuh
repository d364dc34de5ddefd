// qrita_impl.cuh — B200 (sm_100a) exact Top-k / Top-p truncation kernels.
//
// Reference path (arxiv/paper_2602_01518, pkg/src/sigmatop):
//   engine.run_batch (engine.py:82-113) -> pipeline.truncate_topk_topp (pipeline.py:199-239)
//     -> sigma_trunc.{row_stats, lookup_delta_*, threshold_from, gather_outliers, is_hit}
//        (sigma_trunc.py:69-138)
//     -> pivot_search.{quaternary,binary}_{topk,topp} (pivot_search.py:93-244)
//     -> pipeline.finalize_mask / _apply_plan (pipeline.py:47-78)
// Ground truth: oracle.oracle_topk_topp (oracle.py:70-89).
//
// Two pipelines behind one C entry point (DESIGN.md has the full story):
//   qrita_fused  (default; rows 16-byte aligned) one launch, one CTA owns one row at a time, two
//                CTAs per SM, persistent over rows.  The row streams once through a ring of 4 KB
//                shared-memory stages filled by bulk copies (cp.async.bulk + mbarrier); the sigma plan
//                is computed in place from the first stages; outliers are compacted straight into
//                shared memory while the -inf / copy background is written; the row tail (bin-sort
//                resolve, or the pivot searches / distinct-value path on the rare full-row cases)
//                runs in the same CTA on the same shared memory.
//   staged       (unaligned rows, or QRITA_STAGED) qrita_prep -> qrita_stream -> qrita_tail chained
//                with programmatic dependent launch; outliers go through per-row HBM buffers.
// Both share tail_resolve and compute bit-identical results.
//
// Files: qrita_device.cuh (order keys, 192-bit fixed point, mbarrier / bulk-copy primitives),
// qrita_elem.cuh (tables, element / vector access), qrita_plan.cuh (sigma plan, qrita_prep),
// qrita_search.cuh (block primitives, pivot searches), qrita_resolve.cuh (row tail),
// qrita_fused.cuh / qrita_staged.cuh (the two pipelines); this file dispatches between them.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "qrita_types.cuh"
#include "qrita_fused.cuh"
#include "qrita_staged.cuh"
#include "qrita_topp16.cuh"

namespace qrita {

template <typename T>
static cudaError_t launch_all(const Params &P, cudaStream_t st, bool vec, cudaEvent_t prep_done,
                              cudaEvent_t stream_done) {
  // fused single-kernel path: rows and their tail ends must be 16-byte aligned for the bulk copies
  const bool fused_ok = vec && ((size_t)P.V * sizeof(T)) % 16 == 0 && !(P.flags & QRITA_STAGED);
  if (fused_ok) {
    if (prep_done) cudaEventRecord(prep_done, st);
    Params PF = P;
    if constexpr (sizeof(T) == 2) {
      if (P.V >= kStageBytes) {
        // bf16: top-p-only rows go to the two-CTA histogram kernel first; the fused kernel skips them
        cudaError_t e = launch_topp16(P, st);
        if (e != cudaSuccess) return e;
        PF.topp16 = 1;
      }
    }
    const bool pdl = PF.topp16 != 0;
    cudaError_t e = (P.flags & QRITA_SEARCH_BINARY) ? launch_fused<T, 1>(PF, st, pdl) : launch_fused<T, 3>(PF, st, pdl);
    if (e == cudaSuccess && stream_done) e = cudaEventRecord(stream_done, st);
    return e;
  }
  if (P.flags & QRITA_SEARCH_BINARY)
    return vec ? launch_pipeline<T, 1, true>(P, st, prep_done, stream_done)
               : launch_pipeline<T, 1, false>(P, st, prep_done, stream_done);
  return vec ? launch_pipeline<T, 3, true>(P, st, prep_done, stream_done)
             : launch_pipeline<T, 3, false>(P, st, prep_done, stream_done);
}

}  // namespace qrita
