// Definition of scan::launch_nl<NL>; included by exactly one ssb_scan_nl<N>.cu.
#pragma once

#include "ssb_scan.cuh"

namespace laq {
namespace scan {

// variant: 0 = ldg fallback, 1 = TMA pipe, 2 = resident-table stream (int32),
// 3 = the stream kernel over byte-packed columns, 4/5/6 = the direct-probe
// kernel over int32 / byte-packed / bit-packed columns.
template <int NL, int NF, int MODE>
void launch_variant(laq_ctx* ctx, const ScanArgs& a, int variant, bool vec, int grid, size_t smem) {
  cudaStream_t s = ctx->stream;
  const int sm = static_cast<int>(smem);
  if (variant == 1) {
    LAQ_CUDA(cudaFuncSetAttribute(scan_pipe_kernel<NL, NF, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    scan_pipe_kernel<NL, NF, MODE><<<grid, kPipeThreads, smem, s>>>(a);
  } else if (variant >= 4 && variant <= 6) {
    if constexpr (MODE == 2) {
      fail(LAQ_ERR_UNSUPPORTED, "direct scan: global-atomic group mode");
    } else {
      auto kern = variant == 6   ? scan_direct_kernel<NL, NF, MODE, 2>
                  : variant == 5 ? scan_direct_kernel<NL, NF, MODE, 1>
                                 : scan_direct_kernel<NL, NF, MODE, 0>;
      LAQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      const int64_t blocks_needed = (a.n + kDirectThreads * 4 - 1) / (kDirectThreads * 4);
      const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(grid, blocks_needed)));
      kern<<<g, kDirectThreads, smem, s>>>(a);
    }
  } else if (variant == 2 || variant == 3) {
    auto kern = variant == 3 ? scan_stream_kernel<NL, NF, MODE, true> : scan_stream_kernel<NL, NF, MODE, false>;
    LAQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    int per_sm = 0;
    LAQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kStreamThreads, smem));
    const int64_t blocks_needed = (a.n + kStreamThreads * 4 - 1) / (kStreamThreads * 4);
    const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(int64_t{grid} * std::max(per_sm, 1), blocks_needed)));
    kern<<<g, kStreamThreads, smem, s>>>(a);
  } else {
    if (MODE == 1)
      LAQ_CUDA(cudaFuncSetAttribute(scan_ldg_kernel<NL, NF, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    scan_ldg_kernel<NL, NF, MODE><<<grid, 256, MODE == 1 ? smem : 0, s>>>(a, vec);
  }
}

template <int NL, int NF>
void launch_nf(laq_ctx* ctx, const ScanArgs& a, int mode, int variant, bool vec, int grid, size_t smem) {
  if (mode == 0) launch_variant<NL, NF, 0>(ctx, a, variant, vec, grid, smem);
  else if (mode == 1) launch_variant<NL, NF, 1>(ctx, a, variant, vec, grid, smem);
  else launch_variant<NL, NF, 2>(ctx, a, variant, vec, grid, smem);
}

template <int NL>
void launch_nl(laq_ctx* ctx, const ScanArgs& a, int nf, int mode, int variant, bool vec, int grid, size_t smem) {
  switch (nf) {
    case 0: launch_nf<NL, 0>(ctx, a, mode, variant, vec, grid, smem); break;
    case 1: launch_nf<NL, 1>(ctx, a, mode, variant, vec, grid, smem); break;
    case 2: launch_nf<NL, 2>(ctx, a, mode, variant, vec, grid, smem); break;
    case 3: launch_nf<NL, 3>(ctx, a, mode, variant, vec, grid, smem); break;
    case 4: launch_nf<NL, 4>(ctx, a, mode, variant, vec, grid, smem); break;
    default: fail(LAQ_ERR_UNSUPPORTED, "at most 4 fact filters per query");
  }
}

}  // namespace scan
}  // namespace laq

#define LAQ_SCAN_INSTANTIATE(N) \
  template void laq::scan::launch_nl<N>(laq_ctx*, const laq::scan::ScanArgs&, int, int, int, bool, int, size_t);
