// Decision-tree fusion on the device:
//
//   tree_partial     P_j[r, c] = sum_n [B_j[r, col_n] > v_n] H_j[n, c]     fusion.cpp:39-47
//                    (prefuse_tree fusion.cpp:128-144; predict_tree's scores
//                    mlops.cpp:254-268 are the one-"dimension" case over T)
//   apply_fused_tree label[m] = labels[c*] where ((P_0[i_0] + P_1[i_1]) + ...)[c*] == h[c*]
//                    for exactly one leaf c* (fusion.cpp:146-168, mlops.cpp:269-280);
//                    ModelError for the first row matching no leaf or several.
//
// Exactness: the node test is x > v on the dim value itself (the reference's
// dense_times_csr with one 1.0 per node column yields 0 + x*1 = x), and each
// score is the sequential node-order sum 0 + 1*H[n,c] over the nodes whose test
// holds (dense_matmul skips zero entries), so partials and labels are
// bit-identical to the reference for any H.
//
// Layout / kernels: warp per dim row; lanes evaluate 32 nodes at a time and
// ballot the predicate bits into shared memory (p <= 2048 nodes), then each lane
// accumulates leaves c = lane, lane+32, ... over the set bits (uniform across
// the warp: no divergence).  The apply kernel is warp per target row: lanes read
// consecutive leaves of each partial row (coalesced), compare, and a ballot +
// popc decides the unique matching leaf.
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace laq {
namespace tree {

constexpr int kWarps = 8;
constexpr int kMaxNodes = 2048;

__global__ void __launch_bounds__(kWarps * 32) tree_partial_kernel(const double* __restrict__ B, int64_t rows,
                                                                   int64_t cols, int p,
                                                                   const int32_t* __restrict__ node_col,
                                                                   const double* __restrict__ thr,
                                                                   const double* __restrict__ scale,
                                                                   const double* __restrict__ H, int64_t l,
                                                                   double* __restrict__ out) {
  __shared__ uint32_t s_bits[kWarps][kMaxNodes / 32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int words = (p + 31) / 32;
  for (int64_t r = blockIdx.x * (int64_t)kWarps + w; r < rows; r += (int64_t)gridDim.x * kWarps) {
    const double* row = B + r * cols;
    for (int wd = 0; wd < words; ++wd) {
      const int n = wd * 32 + lane;
      bool bit = false;
      if (n < p) {  // a node whose feature this dim does not place reads 0 (empty column of M_j F_j)
        const int32_t nc = __ldg(node_col + n);
        const double x = nc >= 0 ? __dmul_rn(__ldg(row + nc), __ldg(scale + n)) : 0.0;  // 0 + av * v
        bit = x > __ldg(thr + n);
      }
      const uint32_t m = __ballot_sync(0xffffffffu, bit);
      if (lane == 0) s_bits[w][wd] = m;
    }
    __syncwarp();
    for (int64_t c = lane; c < l; c += 32) {
      double acc = 0.0;
      for (int wd = 0; wd < words; ++wd) {
        uint32_t m = s_bits[w][wd];
        while (m) {
          const int n = wd * 32 + __ffs(m) - 1;
          m &= m - 1;
          acc = __dadd_rn(acc, __dmul_rn(1.0, __ldg(H + static_cast<int64_t>(n) * l + c)));
        }
      }
      out[r * l + c] = acc;
    }
    __syncwarp();
  }
}

struct ApplyArgs {
  int n_parts;
  const int64_t* idx[8];  // nullptr = identity
  const double* P[8];
  int64_t rows, l;
  const double* score;   // h (l)
  const int64_t* label;  // (l)
  int64_t* out;
  unsigned long long* bad;  // min over offending rows of (row << 1 | several)
};

__global__ void __launch_bounds__(256) apply_tree_kernel(const ApplyArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t m = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); m < a.rows; m += warps) {
    int64_t src[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < a.n_parts) src[j] = a.idx[j] ? __ldg(a.idx[j] + m) : m;
    int hits = 0, hit = -1;
    for (int64_t c0 = 0; c0 < a.l; c0 += 32) {
      const int64_t c = c0 + lane;
      bool eq = false;
      if (c < a.l) {
        double s = __dadd_rn(0.0, __ldg(a.P[0] + src[0] * a.l + c));  // spmm_dense: 0 + 1*x
#pragma unroll
        for (int j = 1; j < 8; ++j)
          if (j < a.n_parts) s = __dadd_rn(s, __ldg(a.P[j] + src[j] * a.l + c));
        eq = s == __ldg(a.score + c);
      }
      const uint32_t b = __ballot_sync(0xffffffffu, eq);
      if (b && hit < 0) hit = static_cast<int>(c0) + __ffs(b) - 1;
      hits += __popc(b);
    }
    if (lane == 0) {
      if (hits == 1) {
        a.out[m] = __ldg(a.label + hit);
      } else {
        a.out[m] = 0;
        atomicMin(a.bad, (static_cast<unsigned long long>(m) << 1) | (hits > 1 ? 1ull : 0ull));
      }
    }
  }
}

}  // namespace tree
}  // namespace laq

using namespace laq;

extern "C" {

int laq_tree_partial(laq_ctx* ctx, const double* d_B, int64_t rows, int64_t cols, int64_t p,
                     const int64_t* h_node_col, const double* h_node_scale, const double* h_thr,
                     const double* h_path_rows, int64_t l, double* d_out) {
  return guard(ctx, [&] {
    if (p < 0 || l < 0 || rows < 0) fail(LAQ_ERR_SHAPE, "tree_partial: negative size");
    if (p > tree::kMaxNodes) fail(LAQ_ERR_UNSUPPORTED, "tree_partial: more than 2048 nodes in one dimension");
    for (int64_t n = 0; n < p; ++n)
      if (h_node_col[n] < -1 || h_node_col[n] >= cols) fail(LAQ_ERR_SHAPE, "fusion: column map does not fit dim table");
    if (rows == 0 || l == 0) return;
    DevBuf<int32_t> col(ctx, static_cast<size_t>(std::max<int64_t>(p, 1)));
    DevBuf<double> thr(ctx, static_cast<size_t>(std::max<int64_t>(p, 1)));
    DevBuf<double> scl(ctx, static_cast<size_t>(std::max<int64_t>(p, 1)));
    std::vector<double> ones(static_cast<size_t>(p), 1.0);
    DevBuf<double> H(ctx, static_cast<size_t>(std::max<int64_t>(p * l, 1)));
    std::vector<int32_t> c32(h_node_col, h_node_col + p);
    if (p > 0) {
      LAQ_CUDA(cudaMemcpyAsync(col.get(), c32.data(), p * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
      LAQ_CUDA(cudaMemcpyAsync(thr.get(), h_thr, p * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
      LAQ_CUDA(cudaMemcpyAsync(scl.get(), h_node_scale ? h_node_scale : ones.data(), p * sizeof(double),
                               cudaMemcpyHostToDevice, ctx->stream));
      LAQ_CUDA(cudaMemcpyAsync(H.get(), h_path_rows, p * l * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    }
    const int grid = grid_for(rows, tree::kWarps, ctx->sm_count * 8);
    tree::tree_partial_kernel<<<grid, tree::kWarps * 32, 0, ctx->stream>>>(d_B, rows, cols, static_cast<int>(p),
                                                                           col.get(), thr.get(), scl.get(), H.get(), l,
                                                                           d_out);
    launched(ctx);
    sync(ctx);  // host staging vectors must outlive their async copies
  });
}

int laq_apply_fused_tree(laq_ctx* ctx, int32_t n_parts, const int64_t* const* d_idx, int64_t rows,
                         const double* const* d_partials, int64_t l, const double* h_path_score,
                         const int64_t* h_labels, int64_t* d_out, int64_t* h_bad_row, int32_t* h_bad_several) {
  return guard(ctx, [&] {
    if (n_parts < 1 || n_parts > 8) fail(LAQ_ERR_SHAPE, "apply_fused_tree: 1..8 partials");
    *h_bad_row = -1;
    *h_bad_several = 0;
    if (rows == 0) return;
    if (l == 0) {  // every row matches no leaf (fusion.cpp:164)
      *h_bad_row = 0;
      fail(LAQ_ERR_MODEL, "row 0 matches no leaf");
    }
    DevBuf<double> score(ctx, static_cast<size_t>(l));
    DevBuf<int64_t> lab(ctx, static_cast<size_t>(l));
    LAQ_CUDA(cudaMemcpyAsync(score.get(), h_path_score, l * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    LAQ_CUDA(cudaMemcpyAsync(lab.get(), h_labels, l * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    unsigned long long* bad = reinterpret_cast<unsigned long long*>(ctx->d_flags + 59);
    LAQ_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), ctx->stream));
    tree::ApplyArgs a{};
    a.n_parts = n_parts;
    for (int j = 0; j < n_parts; ++j) {
      a.idx[j] = d_idx ? d_idx[j] : nullptr;
      a.P[j] = d_partials[j];
    }
    a.rows = rows;
    a.l = l;
    a.score = score.get();
    a.label = lab.get();
    a.out = d_out;
    a.bad = bad;
    tree::apply_tree_kernel<<<grid_for(rows, 8, ctx->sm_count * 16), 256, 0, ctx->stream>>>(a);
    launched(ctx);
    LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, bad, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    const unsigned long long b = static_cast<unsigned long long>(ctx->h_pinned[0]);
    if (b != ~0ull) {
      *h_bad_row = static_cast<int64_t>(b >> 1);
      *h_bad_several = static_cast<int32_t>(b & 1);
      fail(LAQ_ERR_MODEL, "row " + std::to_string(b >> 1) + ((b & 1) ? " matches several leaves" : " matches no leaf"));
    }
  });
}

}  // extern "C"
