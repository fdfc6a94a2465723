// Definition of scan::launch_nl<NL>; included by exactly one ssb_scan_nl<N>.cu.
#pragma once

#include "ssb_scan.cuh"

namespace laq {
namespace scan {

template <int NL, int NF>
void launch_nf(laq_ctx* ctx, const ScanArgs& a, int mode, bool pipe, bool vec, int grid, size_t smem) {
  cudaStream_t s = ctx->stream;
  const int sm = static_cast<int>(smem);
  if (pipe) {
    if (mode == 0) {
      LAQ_CUDA(cudaFuncSetAttribute(scan_pipe_kernel<NL, NF, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      scan_pipe_kernel<NL, NF, 0><<<grid, kPipeThreads, smem, s>>>(a);
    } else if (mode == 1) {
      LAQ_CUDA(cudaFuncSetAttribute(scan_pipe_kernel<NL, NF, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      scan_pipe_kernel<NL, NF, 1><<<grid, kPipeThreads, smem, s>>>(a);
    } else {
      LAQ_CUDA(cudaFuncSetAttribute(scan_pipe_kernel<NL, NF, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      scan_pipe_kernel<NL, NF, 2><<<grid, kPipeThreads, smem, s>>>(a);
    }
  } else {
    if (mode == 0) {
      scan_ldg_kernel<NL, NF, 0><<<grid, 256, 0, s>>>(a, vec);
    } else if (mode == 1) {
      LAQ_CUDA(cudaFuncSetAttribute(scan_ldg_kernel<NL, NF, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      scan_ldg_kernel<NL, NF, 1><<<grid, 256, smem, s>>>(a, vec);
    } else {
      scan_ldg_kernel<NL, NF, 2><<<grid, 256, 0, s>>>(a, vec);
    }
  }
}

template <int NL>
void launch_nl(laq_ctx* ctx, const ScanArgs& a, int nf, int mode, bool pipe, bool vec, int grid, size_t smem) {
  switch (nf) {
    case 0: launch_nf<NL, 0>(ctx, a, mode, pipe, vec, grid, smem); break;
    case 1: launch_nf<NL, 1>(ctx, a, mode, pipe, vec, grid, smem); break;
    case 2: launch_nf<NL, 2>(ctx, a, mode, pipe, vec, grid, smem); break;
    case 3: launch_nf<NL, 3>(ctx, a, mode, pipe, vec, grid, smem); break;
    case 4: launch_nf<NL, 4>(ctx, a, mode, pipe, vec, grid, smem); break;
    default: fail(LAQ_ERR_UNSUPPORTED, "at most 4 fact filters per query");
  }
}

}  // namespace scan
}  // namespace laq

#define LAQ_SCAN_INSTANTIATE(N) \
  template void laq::scan::launch_nl<N>(laq_ctx*, const laq::scan::ScanArgs&, int, int, bool, bool, int, size_t);
