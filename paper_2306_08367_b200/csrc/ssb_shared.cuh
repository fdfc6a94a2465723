// Shared scan of a batch of queries (ssb_shared.cu): kernel parameters and
// the host launcher used by laq_plans_scan_shared (ssb.cu).
#pragma once

#include "ssb_scan.cuh"

namespace laq {
namespace scan {

constexpr int kMaxShared = 3;

struct SharedScan {
  ScanArgs q[kMaxShared];     // per query: links (smem offsets rebased), filters, bins size, acc
  int64_t bins_off[kMaxShared];  // byte offset of each query's u32 bins
  int64_t flush_every;           // common spill period (min over the queries)
  int prefetch;
};

// nq in {2, 3}; nl 1..4; nf 0..2; mode 0 (one group) or 1 (narrow shared bins).
void launch_shared(laq_ctx* ctx, const SharedScan& M, int nq, int nl, int nf, int mode, size_t smem);

}  // namespace scan
}  // namespace laq
