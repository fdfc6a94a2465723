// Host-side launch of the K4 scan kernels, one explicit instantiation unit per
// link count (ssb_scan_nl<N>.cu) so the 2 x 105 kernel variants compile in
// parallel.
#pragma once

#include "ssb_scan.cuh"

namespace laq {
namespace scan {

template <int NL>
void launch_nl(laq_ctx* ctx, const ScanArgs& a, int nf, int mode, int variant, bool vec, int grid, size_t smem);

#define LAQ_SCAN_EXTERN(N)                                                                                   \
  extern template void launch_nl<N>(laq_ctx*, const ScanArgs&, int, int, int, bool, int, size_t);
LAQ_SCAN_EXTERN(0)
LAQ_SCAN_EXTERN(1)
LAQ_SCAN_EXTERN(2)
LAQ_SCAN_EXTERN(3)
LAQ_SCAN_EXTERN(4)
LAQ_SCAN_EXTERN(5)
LAQ_SCAN_EXTERN(6)
#undef LAQ_SCAN_EXTERN

}  // namespace scan
}  // namespace laq
