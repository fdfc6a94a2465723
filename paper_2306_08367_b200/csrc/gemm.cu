// Dense fp64 contractions: dense_matmul / predict_linear (matrix.cpp:158-174,
// mlops.cpp:248-250) and the pre-fusion prefuse_linear (fusion.cpp:31-36,
// 50-62): P_j = B_j (M_j L).
//
// The reference accumulates every output element as a sequential k-ordered
// sum of separately rounded products (no FMA contraction on x86-64 baseline,
// zero A entries skipped).  This SIMT kernel keeps exactly that order and
// rounding (__dmul_rn then __dadd_rn, k ascending, a == 0 skipped), so the
// device result is bit-identical to the reference; the tile only decides
// which thread owns which outputs.  These are the small GEMMs of the fused
// plan (r_j x k_j x l with small l, HBM/latency-bound); the large tensor-core
// shapes are the separate tcgen05 path.
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace laq {
namespace {

constexpr int TM = 64, TN = 64, TK = 16;  // block tile
constexpr int RM = 4, RN = 4;             // per-thread outputs (16x16 threads)

__global__ void __launch_bounds__(256) dgemm_seq_kernel(const double* __restrict__ A, int64_t m, int64_t k,
                                                        const double* __restrict__ B, int64_t n, double* __restrict__ C) {
  __shared__ double sA[TK][TM + 1];
  __shared__ double sB[TK][TN];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t row0 = blockIdx.x * (int64_t)TM, col0 = blockIdx.y * (int64_t)TN;  // rows on x: no 65535 cap
  double acc[RM][RN];
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN; ++j) acc[i][j] = 0.0;

  for (int64_t k0 = 0; k0 < k; k0 += TK) {
    for (int e = threadIdx.x; e < TM * TK; e += 256) {
      const int r = e / TK, c = e % TK;
      const int64_t gr = row0 + r, gc = k0 + c;
      sA[c][r] = (gr < m && gc < k) ? A[gr * k + gc] : 0.0;
    }
    for (int e = threadIdx.x; e < TK * TN; e += 256) {
      const int r = e / TN, c = e % TN;
      const int64_t gr = k0 + r, gc = col0 + c;
      sB[r][c] = (gr < k && gc < n) ? B[gr * n + gc] : 0.0;
    }
    __syncthreads();
    const int kk = static_cast<int>(std::min<int64_t>(TK, k - k0));
    for (int q = 0; q < kk; ++q) {
      double a[RM], b[RN];
#pragma unroll
      for (int i = 0; i < RM; ++i) a[i] = sA[q][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < RN; ++j) b[j] = sB[q][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < RM; ++i) {
        if (a[i] == 0.0) continue;  // matrix.cpp:168
#pragma unroll
        for (int j = 0; j < RN; ++j) acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(a[i], b[j]));
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN; ++j) {
      const int64_t gr = row0 + ty + 16 * i, gc = col0 + tx + 16 * j;
      if (gr < m && gc < n) C[gr * n + gc] = acc[i][j];
    }
}

// n == 1 (linear regression, l = 1): one warp per row, lanes stride k, then an
// ordered reduction is NOT possible without changing the association -- so each
// thread owns one output row and walks k sequentially (rows are independent).
__global__ void dgemv_seq_kernel(const double* __restrict__ A, int64_t m, int64_t k, const double* __restrict__ B,
                                 double* __restrict__ C) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    const double* a = A + i * k;
    for (int64_t q = 0; q < k; ++q) {
      const double av = a[q];
      if (av == 0.0) continue;
      acc = __dadd_rn(acc, __dmul_rn(av, __ldg(B + q)));
    }
    C[i] = acc;
  }
}

__global__ void gather_rows(const double* __restrict__ L, int64_t l, const int32_t* __restrict__ place, int64_t kj,
                            double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < kj * l; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / l, j = e - c * l;
    out[e] = L[static_cast<int64_t>(place[c]) * l + j];
  }
}

// spmm_dense (matrix.cpp:125-139) for a general CSR: out(i, j) = sum over the
// row's entries, in CSR order, of v * B(col, j) (separately rounded).
__global__ void csr_spmm_dense_kernel(const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ col_idx,
                                      const double* __restrict__ vals, int64_t rows, const double* __restrict__ B,
                                      int64_t n, double* __restrict__ out) {
  const int64_t total = rows * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    double acc = 0.0;
    for (int64_t t = row_ptr[i]; t < row_ptr[i + 1]; ++t) acc = __dadd_rn(acc, __dmul_rn(vals[t], B[col_idx[t] * n + j]));
    out[e] = acc;
  }
}

// materialize's column placement (laqops.cpp:364-371): dst(r, tgt) += v * src(r, src_col).
__global__ void place_columns_kernel(const double* __restrict__ src, int64_t rows, int64_t src_cols,
                                     const int64_t* __restrict__ sc, const int64_t* __restrict__ tc,
                                     const double* __restrict__ v, int64_t nnz, int64_t k, double* __restrict__ dst) {
  const int64_t total = rows * nnz;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / nnz, q = e - r * nnz;
    dst[r * k + tc[q]] = __dadd_rn(dst[r * k + tc[q]], __dmul_rn(v[q], src[r * src_cols + sc[q]]));
  }
}

}  // namespace

void dgemm_seq(laq_ctx* ctx, const double* A, int64_t m, int64_t k, const double* B, int64_t n, double* C) {
  if (m == 0 || n == 0) return;
  if (k == 0) {
    LAQ_CUDA(cudaMemsetAsync(C, 0, m * n * sizeof(double), ctx->stream));
    return;
  }
  if (n == 1) {
    dgemv_seq_kernel<<<grid_for(m, 128, ctx->sm_count * 16), 128, 0, ctx->stream>>>(A, m, k, B, C);
  } else {
    const dim3 grid(static_cast<unsigned>((m + TM - 1) / TM), static_cast<unsigned>((n + TN - 1) / TN));
    if (grid.y > 65535 || (m + TM - 1) / TM > 0x7fffffff) fail(LAQ_ERR_UNSUPPORTED, "dense_matmul: output too wide for one launch");
    dgemm_seq_kernel<<<grid, 256, 0, ctx->stream>>>(A, m, k, B, n, C);
  }
  launched(ctx);
}

}  // namespace laq

using namespace laq;

extern "C" {

int laq_dense_matmul(laq_ctx* ctx, const double* a, int64_t m, int64_t k, const double* b, int64_t n, double* c) {
  return guard(ctx, [&] {
    if (m < 0 || k < 0 || n < 0) fail(LAQ_ERR_SHAPE, "dense_matmul: negative dimension");
    dgemm_seq(ctx, a, m, k, b, n, c);
  });
}

int laq_spmm_dense(laq_ctx* ctx, const int64_t* d_row_ptr, const int64_t* d_col_idx, const double* d_values,
                   int64_t rows, const double* d_b, int64_t b_rows, int64_t n, double* d_out) {
  return guard(ctx, [&] {
    (void)b_rows;
    if (rows == 0 || n == 0) return;
    csr_spmm_dense_kernel<<<grid_for(rows * n, 256, ctx->sm_count * 16), 256, 0, ctx->stream>>>(
        d_row_ptr, d_col_idx, d_values, rows, d_b, n, d_out);
    launched(ctx);
  });
}

int laq_place_columns(laq_ctx* ctx, const double* d_src, int64_t rows, int64_t src_cols, const int64_t* h_src_col,
                      const int64_t* h_tgt_col, const double* h_val, int64_t nnz, int64_t k, double* d_dst) {
  return guard(ctx, [&] {
    if (rows == 0 || nnz == 0) return;
    DevBuf<int64_t> sc(ctx, nnz), tc(ctx, nnz);
    DevBuf<double> v(ctx, nnz);
    LAQ_CUDA(cudaMemcpyAsync(sc.get(), h_src_col, nnz * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    LAQ_CUDA(cudaMemcpyAsync(tc.get(), h_tgt_col, nnz * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    LAQ_CUDA(cudaMemcpyAsync(v.get(), h_val, nnz * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    place_columns_kernel<<<grid_for(rows * nnz, 256, ctx->sm_count * 16), 256, 0, ctx->stream>>>(
        d_src, rows, src_cols, sc.get(), tc.get(), v.get(), nnz, k, d_dst);
    launched(ctx);
    sync(ctx);  // host triplets must outlive the copies
  });
}

int laq_prefuse_linear(laq_ctx* ctx, int32_t n_dims, const double* const* d_dims, const int64_t* h_dim_rows,
                       const int64_t* h_dim_cols, const int64_t* const* h_placements, const double* d_L, int64_t k,
                       int64_t l, double* const* d_partials) {
  return guard(ctx, [&] {
    if (n_dims < 1) fail(LAQ_ERR_SHAPE, "prefuse_linear: dim/map list lengths");
    // check_placements (fusion.cpp:11-25) + make_map target checks (laqops.cpp:33-37).
    std::vector<char> claimed(static_cast<size_t>(k), 0);
    int64_t total = 0;
    for (int j = 0; j < n_dims; ++j)
      for (int64_t c = 0; c < h_dim_cols[j]; ++c) {
        const int64_t t = h_placements[j][c];
        if (t < 0 || t >= k) fail(LAQ_ERR_MAPPING, "column map: target index " + std::to_string(t) + " out of range");
        if (claimed[t]) fail(LAQ_ERR_MAPPING, "fusion: overlapping target column " + std::to_string(t));
        claimed[t] = 1;
        ++total;
      }
    if (total != k)
      fail(LAQ_ERR_SHAPE, "fusion: placements claim " + std::to_string(total) + " of " + std::to_string(k) + " feature columns");
    for (int j = 0; j < n_dims; ++j) {
      const int64_t kj = h_dim_cols[j], rj = h_dim_rows[j];
      // M_j L: the placement picks dim j's row block out of L (exact copies).
      DevBuf<double> ml(ctx, static_cast<size_t>(std::max<int64_t>(kj * l, 1)));
      DevBuf<int32_t> pl(ctx, static_cast<size_t>(std::max<int64_t>(kj, 1)));
      std::vector<int32_t> hp(h_placements[j], h_placements[j] + kj);
      if (kj) {
        LAQ_CUDA(cudaMemcpyAsync(pl.get(), hp.data(), kj * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
        gather_rows<<<grid_for(kj * l, 256, ctx->sm_count * 4), 256, 0, ctx->stream>>>(d_L, l, pl.get(), kj, ml.get());
        launched(ctx);
      }
      dgemm_seq(ctx, d_dims[j], rj, kj, ml.get(), l, d_partials[j]);
      sync(ctx);  // hp must outlive the async copy
    }
  });
}

}  // extern "C"
