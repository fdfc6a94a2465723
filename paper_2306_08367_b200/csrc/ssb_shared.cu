// Shared scan: up to three queries over the same fact columns in ONE pass.
//
// A batch of queries that read the same fact columns in the same roles (the
// same foreign keys, fact filter columns and measure; e.g. Q1.1-Q1.3, or
// Q2.1-Q2.3) is evaluated by one direct-kernel pass: every 16-byte vector of
// every column is loaded once and each query then runs its own filters, probes
// (its own code tables, staged side by side in shared memory) and group bins.
// The queries' arithmetic is unchanged -- only the repeated HBM reads of the
// same columns are shared.  Host side: laq_plans_scan_shared (ssb.cu) checks
// compatibility, aligns each query's link / filter order to the first query's
// columns and rebases the shared-memory offsets; incompatible batches are
// scanned one query at a time.
#include "ssb_shared.cuh"

namespace laq {
namespace scan {

template <int NQ, int NL, int NF, int MODE>
__global__ void __launch_bounds__(kDirectThreads, 1) scan_shared_kernel(const __grid_constant__ SharedScan M) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x;
  // stage every query's compact code tables; zero every query's bins
#pragma unroll
  for (int q = 0; q < NQ; ++q)
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      const LinkProbe& p = M.q[q].link[j];
      if (p.fmt != kFmtGlobal) {
        const uint4* src = static_cast<const uint4*>(p.packed);
        uint4* dst = reinterpret_cast<uint4*>(smem + p.smem_byte);
        for (int w = tid; w < p.smem_bytes / 16; w += kDirectThreads) dst[w] = __ldg(src + w);
      }
    }
  if constexpr (MODE == 1) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      uint32_t* b = reinterpret_cast<uint32_t*>(smem + M.bins_off[q]);
      for (int64_t g = tid; g < 2 * M.q[q].n_groups; g += kDirectThreads) b[g] = 0;
    }
  }
  __syncthreads();

  const uint32_t s_base = smem_u32(smem);
  uint32_t tab_addr[NQ][NL > 0 ? NL : 1];
  uint32_t bins[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    bins[q] = s_base + static_cast<uint32_t>(M.bins_off[q]);
#pragma unroll
    for (int j = 0; j < NL; ++j) tab_addr[q][j] = s_base + static_cast<uint32_t>(M.q[q].link[j].smem_byte);
  }

  const ScanArgs& a = M.q[0];  // column pointers (shared by every query of the batch)
  const int64_t step = static_cast<int64_t>(gridDim.x) * kDirectThreads * 4;
  const int64_t iters = (a.n + step - 1) / step;
  const int64_t full = a.n / step;
  int64_t row0 = (static_cast<int64_t>(blockIdx.x) * kDirectThreads + tid) * 4;
  const bool pf_lane = M.prefetch && (tid & 7) == 0;
  const int64_t pf_rows = static_cast<int64_t>(M.prefetch) * step;

  int4 kvA[NL > 0 ? NL : 1], fvA[NF > 0 ? NF : 1], mvA = make_int4(0, 0, 0, 0);
  int4 kvB[NL > 0 ? NL : 1], fvB[NF > 0 ? NF : 1], mvB = make_int4(0, 0, 0, 0);
  auto load = [&](int4 (&kv)[NL > 0 ? NL : 1], int4 (&fv)[NF > 0 ? NF : 1], int4& mv, int64_t r) {
#pragma unroll
    for (int j = 0; j < NL; ++j) kv[j] = dld<0>(a.fkc[j], r, a.n);
#pragma unroll
    for (int f = 0; f < NF; ++f) fv[f] = dld<0>(a.ffc[f], r, a.n);
    if (a.measure) mv = dld<0>(a.mc, r, a.n);
  };
  load(kvA, fvA, mvA, row0);

  unsigned long long r_cnt[NQ], r_sum[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) r_cnt[q] = r_sum[q] = 0;
  int64_t until_flush = M.flush_every;
  auto one = [&](int64_t it, const int4 (&kv)[NL > 0 ? NL : 1], const int4 (&fv)[NF > 0 ? NF : 1], const int4& mv,
                 int4 (&nkv)[NL > 0 ? NL : 1], int4 (&nfv)[NF > 0 ? NF : 1], int4& nmv) {
    load(nkv, nfv, nmv, row0 + step);
    if (pf_lane && row0 + pf_rows < a.n) {
#pragma unroll
      for (int j = 0; j < NL; ++j) prefetch_l2<0>(a.fkc[j], row0 + pf_rows);
#pragma unroll
      for (int f = 0; f < NF; ++f) prefetch_l2<0>(a.ffc[f], row0 + pf_rows);
      if (a.measure) prefetch_l2<0>(a.mc, row0 + pf_rows);
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      if (it < full) direct_rows<NL, NF, MODE, 0, false>(M.q[q], row0, kv, fv, mv, tab_addr[q], bins[q], r_cnt[q], r_sum[q]);
      else direct_rows<NL, NF, MODE, 0, true>(M.q[q], row0, kv, fv, mv, tab_addr[q], bins[q], r_cnt[q], r_sum[q]);
    }
    if constexpr (MODE == 1) {
      if (--until_flush == 0) {
        until_flush = M.flush_every;
        if (it + 1 < iters) {
          __syncthreads();
#pragma unroll
          for (int q = 0; q < NQ; ++q)
            spill_bins32(reinterpret_cast<uint32_t*>(smem + M.bins_off[q]), M.q[q].n_groups, M.q[q].acc, tid,
                         kDirectThreads);
          __syncthreads();
        }
      }
    }
    row0 += step;
  };
  for (int64_t it = 0; it < iters; it += 2) {
    one(it, kvA, fvA, mvA, kvB, fvB, mvB);
    if (it + 1 < iters) one(it + 1, kvB, fvB, mvB, kvA, fvA, mvA);
  }

  if constexpr (MODE == 0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) flush_single(r_cnt[q], r_sum[q], M.q[q].acc);
  } else {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      spill_bins32(reinterpret_cast<uint32_t*>(smem + M.bins_off[q]), M.q[q].n_groups, M.q[q].acc, tid,
                   kDirectThreads);
  }
}

template <int NQ, int NL, int NF, int MODE>
void launch_shared_t(laq_ctx* ctx, const SharedScan& M, size_t smem) {
  auto kern = scan_shared_kernel<NQ, NL, NF, MODE>;
  LAQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int64_t blocks_needed = (M.q[0].n + kDirectThreads * 4 - 1) / (kDirectThreads * 4);
  const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ctx->sm_count, blocks_needed)));
  kern<<<g, kDirectThreads, smem, ctx->stream>>>(M);
}

template <int NQ, int NL, int NF>
void launch_shared_m(laq_ctx* ctx, const SharedScan& M, int mode, size_t smem) {
  if (mode == 0) launch_shared_t<NQ, NL, NF, 0>(ctx, M, smem);
  else launch_shared_t<NQ, NL, NF, 1>(ctx, M, smem);
}

template <int NQ, int NL>
void launch_shared_f(laq_ctx* ctx, const SharedScan& M, int nf, int mode, size_t smem) {
  switch (nf) {
    case 0: launch_shared_m<NQ, NL, 0>(ctx, M, mode, smem); break;
    case 1: launch_shared_m<NQ, NL, 1>(ctx, M, mode, smem); break;
    case 2: launch_shared_m<NQ, NL, 2>(ctx, M, mode, smem); break;
    default: fail(LAQ_ERR_UNSUPPORTED, "shared scan: at most 2 fact filters");
  }
}

template <int NQ>
void launch_shared_l(laq_ctx* ctx, const SharedScan& M, int nl, int nf, int mode, size_t smem) {
  switch (nl) {
    case 1: launch_shared_f<NQ, 1>(ctx, M, nf, mode, smem); break;
    case 2: launch_shared_f<NQ, 2>(ctx, M, nf, mode, smem); break;
    case 3: launch_shared_f<NQ, 3>(ctx, M, nf, mode, smem); break;
    case 4: launch_shared_f<NQ, 4>(ctx, M, nf, mode, smem); break;
    default: fail(LAQ_ERR_UNSUPPORTED, "shared scan: 1..4 links");
  }
}

void launch_shared(laq_ctx* ctx, const SharedScan& M, int nq, int nl, int nf, int mode, size_t smem) {
  if (nq == 2) launch_shared_l<2>(ctx, M, nl, nf, mode, smem);
  else if (nq == 3) launch_shared_l<3>(ctx, M, nl, nf, mode, smem);
  else fail(LAQ_ERR_UNSUPPORTED, "shared scan: 2 or 3 queries");
  launched(ctx);
}

}  // namespace scan
}  // namespace laq
