// Aggregate-MM: groupby_sum_single (laqops.cpp:376-413) and
// groupby_sum_multi (laqops.cpp:415-455) on the device.
//
// groupby_sum_single = spmm(valued key_matrix(R), key->group matrix) then a
// ones reduction.  The key->group matrix is built as sorted (key, group) runs
// with multiplicities (csr_from_triplets sums duplicates); each R row probes
// its key's run and emits v * multiplicity per group, and every group's terms
// are summed in ascending R-row order (bit-identical to the reference).
//
// groupby_sum_multi = sort-unique over tuples + segmented sum in row order.
// Tuples are ranked per column (distinct values -> dense ranks), packed into
// one mixed-radix code (first column most significant = lexicographic
// order), stably radix-sorted with the row index (only the code's significant
// bits), and every segment is folded sequentially in ascending row order by
// one warp (segsum_kernel) -- the reference's exact accumulation order, so
// fp64 sums are bit-identical.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "probe.cuh"

namespace laq {
namespace {

// Index of v in the sorted distinct array d[0..n) (lower bound); -1 if absent.
__device__ __forceinline__ int64_t find_sorted(const int64_t* __restrict__ d, int64_t n, int64_t v) {
  int64_t a = 0, b = n;
  while (a < b) {
    const int64_t m = (a + b) >> 1;
    if (__ldg(d + m) < v) a = m + 1; else b = m;
  }
  return (a < n && __ldg(d + a) == v) ? a : -1;
}

// Tuple codes for groupby_sum_multi: code[i] = sum over columns of
// rank(col[c][i]) * stride[c] (every value is present in its column's
// distinct array), plus the row index for the stable sort -- all columns in
// one pass (8 B per column in, 16 B out per row).
constexpr int kRankCols = 8;
struct RankArgs {
  int n_cols;
  const int64_t* col[kRankCols];
  const int64_t* distinct[kRankCols];
  int64_t nd[kRankCols], stride[kRankCols];
};

// A column whose values span at most kRankLut gets a shared-memory rank
// table (value - lo -> rank, built per CTA from its distinct array): one
// shared load per row instead of a binary search of dependent L1 loads.
constexpr int kRankLut = 4096;

__global__ void rank_kernel(const __grid_constant__ RankArgs a, int64_t n, int64_t* __restrict__ code,
                            int64_t* __restrict__ row) {
  extern __shared__ int32_t lut[];  // kRankLut entries per column
  uint32_t use_lut = 0;
  int64_t lo[kRankCols];
  for (int k = 0; k < a.n_cols; ++k) {
    lo[k] = a.distinct[k][0];
    if (static_cast<uint64_t>(a.distinct[k][a.nd[k] - 1]) - static_cast<uint64_t>(lo[k]) < kRankLut) {
      use_lut |= 1u << k;
      for (int64_t j = threadIdx.x; j < a.nd[k]; j += blockDim.x)
        lut[k * kRankLut + (a.distinct[k][j] - lo[k])] = static_cast<int32_t>(j);
    }
  }
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = 0;
#pragma unroll 1
    for (int k = 0; k < a.n_cols; ++k) {
      const int64_t v = __ldcs(a.col[k] + i);
      const int64_t r = (use_lut >> k) & 1u ? lut[k * kRankLut + (v - lo[k])] : find_sorted(a.distinct[k], a.nd[k], v);
      c += r * a.stride[k];
    }
    code[i] = c;
    row[i] = i;
  }
}

// Row-ordered segmented sums: segment s = vals[rows[t]] for t in
// [seg_off[s], seg_off[s+1]), folded left to right exactly as the reference's
// sequential loop (laqops.cpp:446-451) -- fp64 addition is not associative,
// so the fold itself stays serial.  One warp per segment: the lanes load 32
// consecutive row ids (coalesced) and gather their values (32 independent
// loads in flight), then lane 0 folds them in order from shuffles.
__global__ void segsum_kernel(const int64_t* __restrict__ seg_off, int64_t n_seg, const int64_t* __restrict__ rows,
                              const double* __restrict__ vals, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = warp; s < n_seg; s += warps) {
    const int64_t b = seg_off[s], e = seg_off[s + 1];
    double acc = 0.0;
    for (int64_t t = b; t < e; t += 32) {
      const int m = e - t < 32 ? static_cast<int>(e - t) : 32;
      const double v = lane < m ? __ldg(vals + rows[t + lane]) : 0.0;
      for (int j = 0; j < m; ++j) {
        const double x = __shfl_sync(0xffffffffu, v, j);
        acc = __dadd_rn(acc, x);
      }
    }
    if (lane == 0) out[s] = acc;
  }
}

__global__ void decode_kernel(const int64_t* __restrict__ codes, int64_t g, const int64_t* __restrict__ distinct,
                              int64_t stride, int64_t range, int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = distinct[(codes[i] / stride) % range];
}

// (key index * G + group index) codes for the S side of groupby_sum_single.
__global__ void pair_code_kernel(const int64_t* __restrict__ ks, const int64_t* __restrict__ gs, int64_t n,
                                 const int64_t* __restrict__ dk, int64_t nk, const int64_t* __restrict__ dg,
                                 int64_t G, int64_t* code) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    code[i] = find_sorted(dk, nk, ks[i]) * G + find_sorted(dg, G, gs[i]);
}

// groupby_sum_single, pass 1: how many (group, value) terms each R row adds
// (its key's number of distinct groups; 0 for a zero value or a key absent from S).
__global__ void single_count(const int64_t* __restrict__ kr, const double* __restrict__ vr, int64_t nr,
                             const int64_t* __restrict__ dk, int64_t nk, const int64_t* __restrict__ key_run_off,
                             int64_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nr; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = 0;
    if (vr[i] != 0.0) {  // key_matrix skips zero values (laqops.cpp:188-190)
      const int64_t kp = find_sorted(dk, nk, kr[i]);
      if (kp >= 0) c = key_run_off[kp + 1] - key_run_off[kp];
    }
    cnt[i] = c;
  }
}

// Pass 2: per_row = spmm(valued key_matrix(R), key->group) entries in R-row
// order: term = v * multiplicity (0.0 + v*m in the reference's accumulator,
// matrix.cpp:107-113, which is exact), tagged with its group.
__global__ void single_terms(const int64_t* __restrict__ kr, const double* __restrict__ vr, int64_t nr,
                             const int64_t* __restrict__ dk, int64_t nk, const int64_t* __restrict__ key_run_off,
                             const int64_t* __restrict__ pair_codes, const int64_t* __restrict__ pair_cnt, int64_t G,
                             const int64_t* __restrict__ row_off, int64_t* __restrict__ term_group,
                             double* __restrict__ term_val, int64_t* __restrict__ term_idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nr; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = vr[i];
    if (v == 0.0) continue;
    const int64_t kp = find_sorted(dk, nk, kr[i]);
    if (kp < 0) continue;
    int64_t o = row_off[i];
    for (int64_t t = key_run_off[kp]; t < key_run_off[kp + 1]; ++t, ++o) {
      term_group[o] = pair_codes[t] % G;
      term_val[o] = __dmul_rn(v, static_cast<double>(pair_cnt[t]));
      term_idx[o] = o;
    }
  }
}

__global__ void scatter_sums(const int64_t* __restrict__ seg_group, const double* __restrict__ seg_sum, int64_t n_seg,
                             double* __restrict__ sums) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n_seg; s += (int64_t)gridDim.x * blockDim.x)
    sums[seg_group[s]] = seg_sum[s];
}

__global__ void key_of_pair(const int64_t* __restrict__ codes, int64_t n, int64_t G, int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = codes[i] / G;
}

__global__ void add_kernel(int64_t* __restrict__ a, const int64_t* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] += b[i];
}

int64_t run_length(laq_ctx* ctx, const int64_t* sorted, int64_t n, int64_t* uniq, int64_t* counts) {
  if (n == 0) return 0;
  int64_t* d_runs = ctx->d_flags + 48;
  size_t b = 0;
  LAQ_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, b, sorted, uniq, counts, d_runs, n, ctx->stream));
  DevBuf<char> tmp(ctx, b);
  LAQ_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.get(), b, sorted, uniq, counts, d_runs, n, ctx->stream));
  ++ctx->launches;
  LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, d_runs, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  return ctx->h_pinned[0];
}

void sort_keys(laq_ctx* ctx, const int64_t* kin, int64_t* kout, int64_t n) {
  if (n == 0) return;
  size_t b = 0;
  LAQ_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, b, kin, kout, n, 0, 64, ctx->stream));
  DevBuf<char> tmp(ctx, b);
  LAQ_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(), b, kin, kout, n, 0, 64, ctx->stream));
  ++ctx->launches;
}

// Stable sort of (key, value) pairs.  max_key >= 0: every key lies in
// [0, max_key], so only its significant bits are sorted (a 7,000-tuple space
// is 13 bits: two onesweep passes instead of eight).
void sort_pairs(laq_ctx* ctx, const int64_t* kin, int64_t* kout, const int64_t* vin, int64_t* vout, int64_t n,
                int64_t max_key = -1) {
  if (n == 0) return;
  const int end_bit = bits_for(max_key);
  size_t b = 0;
  LAQ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, kin, kout, vin, vout, n, 0, end_bit, ctx->stream));
  DevBuf<char> tmp(ctx, b);
  LAQ_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), b, kin, kout, vin, vout, n, 0, end_bit, ctx->stream));
  ++ctx->launches;
}

// Sorted distinct values of a column (signed int64): the bitmap kernels when
// the value range is below 2^31 (group-by columns usually are), else radix
// sort + unique (signed-aware).
int64_t distinct_of(laq_ctx* ctx, const int64_t* col, int64_t n, DevBuf<int64_t>& out) {
  out = DevBuf<int64_t>(ctx, std::max<int64_t>(n, 1));
  if (n == 0) return 0;
  return distinct_sorted(ctx, col, n, nullptr, 0, out.get(), nullptr);
}

}  // namespace
}  // namespace laq

using namespace laq;

extern "C" {

int laq_groupby_sum_single(laq_ctx* ctx, const int64_t* kr, const double* vr, int64_t nr, const int64_t* ks,
                           const int64_t* gs, int64_t ns, int64_t* out_groups, double* out_sums, int64_t* h_n) {
  return guard(ctx, [&] {
    // build_key_domain(keys_r, keys_s): negative keys are a DomainError.
    int64_t mn, mx;
    if (nr) { minmax_i64(ctx, kr, nr, &mn, &mx); if (mn < 0) fail(LAQ_ERR_DOMAIN, "negative join key " + std::to_string(mn)); }
    if (ns) { minmax_i64(ctx, ks, ns, &mn, &mx); if (mn < 0) fail(LAQ_ERR_DOMAIN, "negative join key " + std::to_string(mn)); }
    // Groups: distinct group_s ascending (laqops.cpp:385-387).
    DevBuf<int64_t> groups, dkeys;
    const int64_t G = distinct_of(ctx, gs, ns, groups);
    *h_n = G;
    if (G == 0) return;
    const int64_t NK = distinct_of(ctx, ks, ns, dkeys);
    if (NK > 0 && G > INT64_MAX / NK) fail(LAQ_ERR_UNSUPPORTED, "groupby_sum_single: key x group space overflows");
    // key->group matrix with multiplicities (csr_from_triplets sums duplicates).
    DevBuf<int64_t> codes(ctx, ns), sorted(ctx, ns), uniq(ctx, ns), cnt(ctx, ns);
    const int g = ctx->sm_count * 8;
    pair_code_kernel<<<grid_for(ns, 256, g), 256, 0, ctx->stream>>>(ks, gs, ns, dkeys.get(), NK, groups.get(), G,
                                                                    codes.get());
    launched(ctx);
    sort_keys(ctx, codes.get(), sorted.get(), ns);
    const int64_t npairs = run_length(ctx, sorted.get(), ns, uniq.get(), cnt.get());
    // Per key index: the range of its (group, multiplicity) pairs.
    DevBuf<int64_t> kop(ctx, npairs), kuniq(ctx, npairs), kcnt(ctx, npairs), key_off(ctx, NK + 1);
    key_of_pair<<<grid_for(npairs, 256, g), 256, 0, ctx->stream>>>(uniq.get(), npairs, G, kop.get());
    launched(ctx);
    const int64_t nk2 = run_length(ctx, kop.get(), npairs, kuniq.get(), kcnt.get());
    if (nk2 != NK) fail(LAQ_ERR_GENERIC, "groupby_sum_single: key runs mismatch");
    int64_t total = 0;
    exclusive_scan_i64(ctx, kcnt.get(), key_off.get(), NK, &total);
    ctx->h_pinned[8] = total;
    LAQ_CUDA(cudaMemcpyAsync(key_off.get() + NK, &ctx->h_pinned[8], sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    LAQ_CUDA(cudaMemsetAsync(out_sums, 0, G * sizeof(double), ctx->stream));
    if (nr) {
      // The ones reduction sums per_row's entries in ascending R-row order
      // (laqops.cpp:404-405): terms are laid out in row order, stably sorted
      // by group, and each group's run is summed sequentially (segsum_kernel).
      DevBuf<int64_t> rcnt(ctx, nr), roff(ctx, nr);
      single_count<<<grid_for(nr, 256, g), 256, 0, ctx->stream>>>(kr, vr, nr, dkeys.get(), NK, key_off.get(),
                                                                  rcnt.get());
      launched(ctx);
      int64_t nt = 0;
      exclusive_scan_i64(ctx, rcnt.get(), roff.get(), nr, &nt);
      if (nt > 0) {
        DevBuf<int64_t> tg(ctx, nt), ti(ctx, nt), sg(ctx, nt), si(ctx, nt), ug(ctx, nt), uc(ctx, nt), so(ctx, nt + 1);
        DevBuf<double> tv(ctx, nt), ss(ctx, nt);
        single_terms<<<grid_for(nr, 256, g), 256, 0, ctx->stream>>>(kr, vr, nr, dkeys.get(), NK, key_off.get(),
                                                                    uniq.get(), cnt.get(), G, roff.get(), tg.get(),
                                                                    tv.get(), ti.get());
        launched(ctx);
        sort_pairs(ctx, tg.get(), sg.get(), ti.get(), si.get(), nt, G - 1);  // stable: row order kept per group
        const int64_t ng = run_length(ctx, sg.get(), nt, ug.get(), uc.get());
        int64_t tot = 0;
        exclusive_scan_i64(ctx, uc.get(), so.get(), ng, &tot);
        ctx->h_pinned[8] = tot;
        LAQ_CUDA(cudaMemcpyAsync(so.get() + ng, &ctx->h_pinned[8], sizeof(int64_t), cudaMemcpyHostToDevice,
                                 ctx->stream));
        segsum_kernel<<<grid_for(32 * ng, 256, g), 256, 0, ctx->stream>>>(so.get(), ng, si.get(), tv.get(), ss.get());
        launched(ctx);
        scatter_sums<<<grid_for(ng, 256, g), 256, 0, ctx->stream>>>(ug.get(), ss.get(), ng, out_sums);
        launched(ctx);
      }
    }
    LAQ_CUDA(cudaMemcpyAsync(out_groups, groups.get(), G * sizeof(int64_t), cudaMemcpyDeviceToDevice, ctx->stream));
    sync(ctx);
  });
}

int laq_groupby_sum_multi(laq_ctx* ctx, int32_t n_cols, const int64_t* const* d_cols, const double* d_vals, int64_t n,
                          int64_t* d_out_keys, double* d_out_sums, int64_t capacity, int64_t* h_n_groups) {
  return guard(ctx, [&] {
    if (n_cols < 1) fail(LAQ_ERR_SHAPE, "groupby_sum_multi: no group columns");
    *h_n_groups = 0;
    if (n == 0) return;
    const int g = ctx->sm_count * 8;
    std::vector<DevBuf<int64_t>> distinct(n_cols);
    std::vector<int64_t> nd(n_cols), stride(n_cols);
    for (int c = 0; c < n_cols; ++c) nd[c] = distinct_of(ctx, d_cols[c], n, distinct[c]);
    int64_t s = 1;
    for (int c = n_cols - 1; c >= 0; --c) {
      stride[c] = s;
      if (s > (INT64_MAX / 2) / nd[c]) fail(LAQ_ERR_UNSUPPORTED, "groupby_sum_multi: tuple space exceeds 2^62");
      s *= nd[c];
    }
    DevBuf<int64_t> code(ctx, n), iota(ctx, n), scode(ctx, n), srow(ctx, n);
    for (int c0 = 0; c0 < n_cols; c0 += kRankCols) {  // > 8 columns: accumulate over several passes
      RankArgs ra{};
      ra.n_cols = std::min(kRankCols, n_cols - c0);
      for (int k = 0; k < ra.n_cols; ++k) {
        ra.col[k] = d_cols[c0 + k];
        ra.distinct[k] = distinct[c0 + k].get();
        ra.nd[k] = nd[c0 + k];
        ra.stride[k] = stride[c0 + k];
      }
      const size_t lut = static_cast<size_t>(ra.n_cols) * kRankLut * sizeof(int32_t);
      LAQ_CUDA(cudaFuncSetAttribute(rank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(lut)));
      const int rg = grid_for(n, 512, ctx->sm_count * 4);
      if (c0 == 0) {
        rank_kernel<<<rg, 512, lut, ctx->stream>>>(ra, n, code.get(), iota.get());
      } else {
        DevBuf<int64_t> part(ctx, n);
        rank_kernel<<<rg, 512, lut, ctx->stream>>>(ra, n, part.get(), iota.get());
        add_kernel<<<grid_for(n, 256, g), 256, 0, ctx->stream>>>(code.get(), part.get(), n);
        launched(ctx);
      }
      launched(ctx);
    }
    // Stable: rows stay ascending within a tuple (laqops.cpp:424-429).
    sort_pairs(ctx, code.get(), scode.get(), iota.get(), srow.get(), n, s - 1);
    DevBuf<int64_t> uniq(ctx, n), cnt(ctx, n), off(ctx, n + 1);
    const int64_t G = run_length(ctx, scode.get(), n, uniq.get(), cnt.get());
    if (G > capacity) fail(LAQ_ERR_CAPACITY, "groupby_sum_multi: output capacity");
    int64_t total = 0;
    exclusive_scan_i64(ctx, cnt.get(), off.get(), G, &total);
    ctx->h_pinned[8] = total;
    LAQ_CUDA(cudaMemcpyAsync(off.get() + G, &ctx->h_pinned[8], sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    segsum_kernel<<<grid_for(32 * G, 256, g), 256, 0, ctx->stream>>>(off.get(), G, srow.get(), d_vals, d_out_sums);
    launched(ctx);
    for (int c = 0; c < n_cols; ++c) {
      decode_kernel<<<grid_for(G, 256, g), 256, 0, ctx->stream>>>(uniq.get(), G, distinct[c].get(), stride[c], nd[c],
                                                                 d_out_keys + c * capacity);
      launched(ctx);
    }
    sync(ctx);
    *h_n_groups = G;
  });
}

}  // extern "C"
