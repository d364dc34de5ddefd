// qrita_internal.h — library-internal entry points shared between the C-ABI translation units.
#pragma once
#include <stddef.h>
#include <stdint.h>

#include "qrita_b200.h"

namespace qrita {

// qrita_topk_topp_ex / _idx with the status and nf_col words optionally outside the workspace, and
// kept_idx with any leading dimension the caller can guarantee (kept <= ld_idx per row).
int topk_topp_impl(const void *logits, int64_t ld_in, int dtype, int B, int V, const int64_t *k, const double *p,
                   void *out, int64_t ld_out, int32_t *kept_count, qrita_row_metrics *metrics, void *workspace,
                   size_t ws_bytes, int flags, int sample_size, qrita_stream_t stream, void *prep_done_event,
                   void *stream_done_event, int32_t *status, int32_t *nf_col, int32_t *kept_idx = nullptr,
                   int64_t ld_idx = 0);

}  // namespace qrita
