// The rest of the reference's matrix / selection API on the device:
//
//   check_canonical(SparseCoo)  matrix.cpp:243-255   laq_coo_check
//   csr_from_coo                matrix.cpp:210-221   laq_csr_from_coo
//   coo_from_csr                matrix.cpp:198-208   laq_coo_from_csr
//   spmm (Gustavson SpGEMM)     matrix.cpp:81-123    laq_spmm
//   build_selection_mask /      laqops.cpp:65-85     laq_selection_mask
//     Predicate::matches        predicate.hpp:81-103
//   mask_and                    laqops.cpp:87-93     laq_mask_and
//   apply_mask (Table/DenseMat) laqops.cpp:95-121    laq_mask_indices + laq_gather
//   sort_rows                   laqops.cpp:457-478   laq_sort_rows
//   to_matrix + spmm_dense(I)   cli.cpp:96-101       laq_gather (one-hot row gather, exact)
//   column_to_ints              cli.cpp:65-69        laq_gather (llround)
//   dense_matmul(ones, v)       cli.cpp:103-107      laq_sum_f64
//
// All HBM-bound integer / byte work: one pass per operand,
// grid-stride kernels sized to the SM count; sorts are CUB's onesweep radix
// sort (stable, so the reference's tie orders survive).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace laq {
namespace {

constexpr int kT = 256;

inline int blocks(laq_ctx* ctx, int64_t n) { return grid_for(n, kT, ctx->sm_count * 8); }

// ---- canonical COO check (matrix.cpp:243-255): first failing entry ---------
__global__ void coo_check_kernel(const int64_t* __restrict__ r, const int64_t* __restrict__ c, int64_t nnz,
                                 int64_t rows, int64_t cols, unsigned long long* first_bad) {
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < nnz; m += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rm = r[m], cm = c[m];
    bool bad = rm < 0 || rm >= rows || cm < 0 || cm >= cols;
    if (!bad && m > 0) {
      const int64_t rp = r[m - 1], cp = c[m - 1];
      bad = !(rm > rp || (rm == rp && cm > cp));
    }
    if (bad) atomicMin(first_bad, static_cast<unsigned long long>(m));
  }
}

// row_ptr[i] = lower_bound(row_idx, i) over a row-sorted COO (csr_from_coo's counts + prefix sum).
__global__ void row_ptr_kernel(const int64_t* __restrict__ r, int64_t nnz, int64_t rows, int64_t* __restrict__ rp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= rows; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = 0, b = nnz;
    while (a < b) {
      const int64_t mid = (a + b) >> 1;
      if (__ldg(r + mid) < i) a = mid + 1; else b = mid;
    }
    rp[i] = a;
  }
}

// row_idx[e] = the row whose [row_ptr[i], row_ptr[i+1]) holds e (coo_from_csr).
__global__ void expand_rows_kernel(const int64_t* __restrict__ rp, int64_t rows, int64_t nnz, int64_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = 0, b = rows;  // last i with rp[i] <= e
    while (a < b) {
      const int64_t mid = (a + b + 1) >> 1;
      if (__ldg(rp + mid) <= e) a = mid; else b = mid - 1;
    }
    out[e] = a;
  }
}

void coo_check(laq_ctx* ctx, const int64_t* r, const int64_t* c, int64_t nnz, int64_t rows, int64_t cols) {
  if (rows < 0 || cols < 0) fail(LAQ_ERR_GENERIC, "coo: negative dimension");
  if (nnz == 0) return;
  unsigned long long* bad = reinterpret_cast<unsigned long long*>(ctx->d_flags + 60);
  LAQ_CUDA(cudaMemsetAsync(bad, 0xFF, sizeof(unsigned long long), ctx->stream));
  coo_check_kernel<<<blocks(ctx, nnz), kT, 0, ctx->stream>>>(r, c, nnz, rows, cols, bad);
  launched(ctx);
  LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, bad, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  const unsigned long long m = static_cast<unsigned long long>(ctx->h_pinned[0]);
  if (m == ~0ull) return;
  int64_t rc[2];
  LAQ_CUDA(cudaMemcpy(&rc[0], r + m, sizeof(int64_t), cudaMemcpyDeviceToHost));
  LAQ_CUDA(cudaMemcpy(&rc[1], c + m, sizeof(int64_t), cudaMemcpyDeviceToHost));
  if (rc[0] < 0 || rc[0] >= rows || rc[1] < 0 || rc[1] >= cols) fail(LAQ_ERR_GENERIC, "coo: entry out of bounds");
  fail(LAQ_ERR_GENERIC, "coo: entries not sorted or duplicated");
}

// ---- spmm (matrix.cpp:81-123) -----------------------------------------------
__global__ void spmm_count_kernel(const int64_t* __restrict__ a_ci, int64_t a_nnz, const int64_t* __restrict__ b_rp,
                                  int64_t b_rows, int64_t* __restrict__ cnt, int* bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < a_nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = a_ci[e];
    if (k < 0 || k >= b_rows) {
      atomicOr(bad, 1);
      cnt[e] = 0;
    } else {
      cnt[e] = b_rp[k + 1] - b_rp[k];
    }
  }
}

// Every product a(i,k) * b(k,j), in the reference's accumulation order: A's
// entries of row i in CSR order, then B's row k in CSR order.  The products of
// one A entry go to [off[e], off[e] + cnt[e]); the key is (i, j) row-major.
__global__ void spmm_expand_kernel(const int64_t* __restrict__ a_row, const int64_t* __restrict__ a_ci,
                                   const double* __restrict__ a_v, int64_t a_nnz, const int64_t* __restrict__ b_rp,
                                   const int64_t* __restrict__ b_ci, const double* __restrict__ b_v, int64_t b_cols,
                                   const int64_t* __restrict__ off, uint64_t* __restrict__ key,
                                   double* __restrict__ val, int64_t* __restrict__ idx) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < a_nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = a_ci[e];
    const double av = a_v[e];
    const uint64_t base = static_cast<uint64_t>(a_row[e]) * static_cast<uint64_t>(b_cols);
    int64_t o = off[e];
    for (int64_t kk = b_rp[k]; kk < b_rp[k + 1]; ++kk, ++o) {
      key[o] = base + static_cast<uint64_t>(b_ci[kk]);
      val[o] = __dmul_rn(av, b_v[kk]);
      idx[o] = o;
    }
  }
}

// acc = 0.0; acc += product, sequentially in the reference's order (matrix.cpp:106-113).
__global__ void segsum_seq_kernel(const int64_t* __restrict__ seg_off, int64_t n_seg, const int64_t* __restrict__ order,
                                  const double* __restrict__ val, double* __restrict__ out, uint8_t* __restrict__ keep) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n_seg; s += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t t = seg_off[s]; t < seg_off[s + 1]; ++t) acc = __dadd_rn(acc, __ldg(val + order[t]));
    out[s] = acc;
    keep[s] = acc != 0.0;  // matrix.cpp:117: exact zeros are not stored
  }
}

__global__ void spmm_emit_kernel(const int64_t* __restrict__ pos, int64_t n, const uint64_t* __restrict__ key,
                                 const double* __restrict__ sum, int64_t b_cols, int64_t* __restrict__ out_row,
                                 int64_t* __restrict__ out_ci, double* __restrict__ out_v) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = pos[t];
    const uint64_t k = key[s];
    out_row[t] = static_cast<int64_t>(k / static_cast<uint64_t>(b_cols));
    out_ci[t] = static_cast<int64_t>(k % static_cast<uint64_t>(b_cols));
    out_v[t] = sum[s];
  }
}

// ---- selection masks (laqops.cpp:65-85, predicate.hpp:81-103) ---------------
template <class T>
__device__ __forceinline__ bool pred_eval(int kind, T v, T lo, T hi, const T* __restrict__ set, int64_t n) {
  switch (kind) {
    case LAQ_PRED_LT: return v < lo;
    case LAQ_PRED_LE: return v <= lo;
    case LAQ_PRED_EQ: return v == lo;
    case LAQ_PRED_GE: return v >= lo;
    case LAQ_PRED_GT: return v > lo;
    case LAQ_PRED_BETWEEN: return v >= lo && v <= hi;
    default: {  // std::binary_search over the sorted set: lower_bound with <, then !(v < *it)
      int64_t a = 0, b = n;
      while (a < b) {
        const int64_t m = (a + b) >> 1;
        if (set[m] < v) a = m + 1; else b = m;
      }
      return a < n && !(v < set[a]);
    }
  }
}

template <class T>
__global__ void mask_kernel(const T* __restrict__ col, int64_t n, int kind, T lo, T hi, const T* __restrict__ set,
                            int64_t set_n, uint8_t* __restrict__ mask, int and_into) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const bool m = pred_eval<T>(kind, col[i], lo, hi, set, set_n);
    mask[i] = and_into ? static_cast<uint8_t>(mask[i] && m) : static_cast<uint8_t>(m);
  }
}

__global__ void mask_and_kernel(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, int64_t n,
                                uint8_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = static_cast<uint8_t>(a[i] && b[i]);
}

// Positions of the set entries, ascending (the order apply_mask keeps): warp
// ballot + per-block offsets from a scan of block counts.
__global__ void mask_count_kernel(const uint8_t* __restrict__ mask, int64_t n, int64_t per_block, int64_t* cnt) {
  const int64_t b0 = blockIdx.x * per_block, b1 = min(n, b0 + per_block);
  int64_t c = 0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) c += mask[i] != 0;
  c = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(c));
  __shared__ int64_t part[kT / 32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < kT / 32; ++w) t += part[w];
    cnt[blockIdx.x] = t;
  }
}

__global__ void mask_emit_kernel(const uint8_t* __restrict__ mask, int64_t n, int64_t per_block,
                                 const int64_t* __restrict__ off, int64_t* __restrict__ out) {
  __shared__ int64_t base;
  __shared__ int warp_cnt[kT / 32];
  const int64_t b0 = blockIdx.x * per_block, b1 = min(n, b0 + per_block);
  if (threadIdx.x == 0) base = off[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t s = b0; s < b1; s += kT) {
    const int64_t i = s + threadIdx.x;
    const bool m = i < b1 && mask[i];
    const unsigned bal = __ballot_sync(0xffffffffu, m);
    if (lane == 0) warp_cnt[warp] = __popc(bal);
    __syncthreads();
    int64_t before = base;
    for (int w = 0; w < warp; ++w) before += warp_cnt[w];
    if (m) out[before + __popc(bal & ((1u << lane) - 1))] = i;
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t t = 0;
      for (int w = 0; w < kT / 32; ++w) t += warp_cnt[w];
      base += t;
    }
    __syncthreads();
  }
}

// ---- gathers (apply_mask, to_matrix + one-hot spmm_dense, column_to_ints) ---
// src kinds: 0 int32, 1 int64, 2 double.  out kinds: 1 int64 (exact copy),
// 2 double ((double) v: to_matrix, storage.cpp), 3 llround((double) v).
__global__ void gather_kernel(const void* __restrict__ src, int src_kind, int64_t row_elems,
                              const int64_t* __restrict__ idx, int64_t n, void* __restrict__ dst, int out_kind) {
  const int64_t total = n * row_elems;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / row_elems, c = t - r * row_elems;
    const int64_t s = (idx ? idx[r] : r) * row_elems + c;
    if (out_kind == 1) {
      static_cast<int64_t*>(dst)[t] = src_kind == 0 ? static_cast<const int32_t*>(src)[s]
                                                    : static_cast<const int64_t*>(src)[s];
      continue;
    }
    double v;
    if (src_kind == 0) v = static_cast<double>(static_cast<const int32_t*>(src)[s]);
    else if (src_kind == 1) v = static_cast<double>(static_cast<const int64_t*>(src)[s]);
    else v = static_cast<const double*>(src)[s];
    if (out_kind == 2) static_cast<double*>(dst)[t] = v;
    else static_cast<int64_t*>(dst)[t] = llround(v);
  }
}

// ---- sums (dense_matmul(ones, v), matrix.cpp:158-174) -----------------------
__global__ void integral_check_kernel(const double* __restrict__ v, int64_t n, double limit, int* not_exact) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = v[i];
    if (!(fabs(x) <= limit) || x != trunc(x)) atomicOr(not_exact, 1);
  }
}

__global__ void sum_i64_kernel(const double* __restrict__ v, int64_t n, unsigned long long* out) {
  int64_t s = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += static_cast<int64_t>(v[i]);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, static_cast<unsigned long long>(s));
}

// The reference's order exactly: dst = 0.0; dst += 1.0 * v[i] for i ascending.
__global__ void sum_seq_kernel(const double* __restrict__ v, int64_t n, double* out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc = __dadd_rn(acc, v[i]);
  *out = acc;
}

// ---- sort_rows (laqops.cpp:457-478) ----------------------------------------
// A total order on doubles that agrees with < on every non-NaN pair and calls
// -0.0 and 0.0 equal (the reference compares with != and <).
__global__ void sort_key_kernel(const double* __restrict__ t, int64_t cols, int64_t col, const int64_t* __restrict__ perm,
                                int64_t rows, int desc, uint64_t* __restrict__ key) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x) {
    double x = t[perm[i] * cols + col];
    if (x == 0.0) x = 0.0;
    if (x != x) x = __longlong_as_double(0x7ff8000000000000ll);
    uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
    b = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    key[i] = desc ? ~b : b;
  }
}

__global__ void iota_kernel(int64_t* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) out[i] = i;
}

template <class K>
void sort_pairs(laq_ctx* ctx, const K* kin, K* kout, const int64_t* vin, int64_t* vout, int64_t n, int end_bit) {
  if (n == 0) return;
  size_t b = 0;
  LAQ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, kin, kout, vin, vout, n, 0, end_bit, ctx->stream));
  DevBuf<char> tmp(ctx, b);
  LAQ_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), b, kin, kout, vin, vout, n, 0, end_bit, ctx->stream));
  ++ctx->launches;
}

int64_t mask_positions(laq_ctx* ctx, const uint8_t* mask, int64_t n, int64_t* out) {
  if (n == 0) return 0;
  const int64_t per_block = 16 * kT;
  const int64_t nb = (n + per_block - 1) / per_block;
  DevBuf<int64_t> cnt(ctx, nb);
  mask_count_kernel<<<static_cast<unsigned>(nb), kT, 0, ctx->stream>>>(mask, n, per_block, cnt.get());
  launched(ctx);
  int64_t total = 0;
  exclusive_scan_i64(ctx, cnt.get(), cnt.get(), nb, &total);
  if (out && total) {
    mask_emit_kernel<<<static_cast<unsigned>(nb), kT, 0, ctx->stream>>>(mask, n, per_block, cnt.get(), out);
    launched(ctx);
  }
  return total;
}

}  // namespace
}  // namespace laq

using namespace laq;

extern "C" {

int laq_coo_check(laq_ctx* ctx, const int64_t* d_row_idx, const int64_t* d_col_idx, int64_t nnz, int64_t rows,
                  int64_t cols) {
  return guard(ctx, [&] { coo_check(ctx, d_row_idx, d_col_idx, nnz, rows, cols); });
}

int laq_csr_from_coo(laq_ctx* ctx, const int64_t* d_row_idx, const int64_t* d_col_idx, int64_t nnz, int64_t rows,
                     int64_t cols, int64_t* d_row_ptr) {
  return guard(ctx, [&] {
    coo_check(ctx, d_row_idx, d_col_idx, nnz, rows, cols);
    row_ptr_kernel<<<blocks(ctx, rows + 1), kT, 0, ctx->stream>>>(d_row_idx, nnz, rows, d_row_ptr);
    launched(ctx);
  });
}

int laq_coo_from_csr(laq_ctx* ctx, const int64_t* d_row_ptr, int64_t rows, int64_t nnz, int64_t* d_row_idx) {
  return guard(ctx, [&] {
    if (nnz <= 0) return;
    expand_rows_kernel<<<blocks(ctx, nnz), kT, 0, ctx->stream>>>(d_row_ptr, rows, nnz, d_row_idx);
    launched(ctx);
  });
}

int laq_spmm(laq_ctx* ctx, const int64_t* a_rp, const int64_t* a_ci, const double* a_v, int64_t a_rows, int64_t a_cols,
             const int64_t* b_rp, const int64_t* b_ci, const double* b_v, int64_t b_rows, int64_t b_cols,
             int64_t* d_c_rp, int64_t* d_c_ci, double* d_c_v, int64_t capacity, int64_t* h_nnz) {
  return guard(ctx, [&] {
    if (a_cols != b_rows) fail(LAQ_ERR_SHAPE, "spmm: shape mismatch");
    *h_nnz = 0;
    int64_t a_nnz = 0;
    if (a_rows > 0) {
      LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, a_rp + a_rows, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
      sync(ctx);
      a_nnz = ctx->h_pinned[0];
    }
    auto zero_rows = [&] {
      if (a_rows >= 0) LAQ_CUDA(cudaMemsetAsync(d_c_rp, 0, (a_rows + 1) * sizeof(int64_t), ctx->stream));
    };
    if (a_nnz == 0 || b_cols == 0) { zero_rows(); return; }
    if (static_cast<double>(a_rows) * static_cast<double>(b_cols) >= 9.2e18)
      fail(LAQ_ERR_UNSUPPORTED, "spmm: rows x cols exceeds 2^63");
    // products per A entry -> offsets
    DevBuf<int64_t> cnt(ctx, a_nnz), arow(ctx, a_nnz);
    int* bad = reinterpret_cast<int*>(ctx->d_flags + 61);
    LAQ_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
    spmm_count_kernel<<<blocks(ctx, a_nnz), kT, 0, ctx->stream>>>(a_ci, a_nnz, b_rp, b_rows, cnt.get(), bad);
    launched(ctx);
    int64_t P = 0;
    exclusive_scan_i64(ctx, cnt.get(), cnt.get(), a_nnz, &P);
    LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    if (*reinterpret_cast<int*>(ctx->h_pinned)) fail(LAQ_ERR_INDEX, "spmm: column index out of range");
    if (P == 0) { zero_rows(); return; }
    expand_rows_kernel<<<blocks(ctx, a_nnz), kT, 0, ctx->stream>>>(a_rp, a_rows, a_nnz, arow.get());
    launched(ctx);
    DevBuf<uint64_t> key(ctx, P), skey(ctx, P);
    DevBuf<double> val(ctx, P);
    DevBuf<int64_t> idx(ctx, P), sidx(ctx, P);
    spmm_expand_kernel<<<blocks(ctx, a_nnz), kT, 0, ctx->stream>>>(arow.get(), a_ci, a_v, a_nnz, b_rp, b_ci, b_v, b_cols,
                                                                  cnt.get(), key.get(), val.get(), idx.get());
    launched(ctx);
    const uint64_t maxkey = static_cast<uint64_t>(a_rows) * static_cast<uint64_t>(b_cols);
    const int end_bit = std::max(1, 64 - __builtin_clzll(maxkey));
    sort_pairs<uint64_t>(ctx, key.get(), skey.get(), idx.get(), sidx.get(), P, end_bit);  // stable
    // runs of equal (i, j)
    DevBuf<uint64_t> ukey(ctx, P);
    DevBuf<int64_t> ucnt(ctx, P), uoff(ctx, P + 1);
    int64_t* d_runs = ctx->d_flags + 62;
    size_t b = 0;
    LAQ_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, b, skey.get(), ukey.get(), ucnt.get(), d_runs, P, ctx->stream));
    {
      DevBuf<char> tmp(ctx, b);
      LAQ_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.get(), b, skey.get(), ukey.get(), ucnt.get(), d_runs, P,
                                                  ctx->stream));
      ++ctx->launches;
    }
    LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, d_runs, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    const int64_t U = ctx->h_pinned[0];
    int64_t tot = 0;
    exclusive_scan_i64(ctx, ucnt.get(), uoff.get(), U, &tot);
    ctx->h_pinned[8] = tot;
    LAQ_CUDA(cudaMemcpyAsync(uoff.get() + U, &ctx->h_pinned[8], sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    DevBuf<double> usum(ctx, U);
    DevBuf<uint8_t> keep(ctx, U);
    segsum_seq_kernel<<<blocks(ctx, U), kT, 0, ctx->stream>>>(uoff.get(), U, sidx.get(), val.get(), usum.get(),
                                                             keep.get());
    launched(ctx);
    DevBuf<int64_t> pos(ctx, U);
    const int64_t nnz = mask_positions(ctx, keep.get(), U, pos.get());
    *h_nnz = nnz;
    if (nnz > capacity) fail(LAQ_ERR_CAPACITY, "spmm: output capacity");
    DevBuf<int64_t> crow(ctx, std::max<int64_t>(nnz, 1));
    if (nnz) {
      spmm_emit_kernel<<<blocks(ctx, nnz), kT, 0, ctx->stream>>>(pos.get(), nnz, ukey.get(), usum.get(), b_cols,
                                                                 crow.get(), d_c_ci, d_c_v);
      launched(ctx);
    }
    row_ptr_kernel<<<blocks(ctx, a_rows + 1), kT, 0, ctx->stream>>>(crow.get(), nnz, a_rows, d_c_rp);
    launched(ctx);
    sync(ctx);
  });
}

int laq_selection_mask(laq_ctx* ctx, const void* d_col, int32_t col_is_float, int64_t n, const laq_pred* p,
                       uint8_t* d_mask, int32_t and_into) {
  return guard(ctx, [&] {
    if (n == 0) return;  // Predicate::matches is never called: no TypeError on an empty column
    if (p->is_float && !col_is_float) fail(LAQ_ERR_TYPE, "predicate constant is float, column is integer");
    if (!p->is_float && col_is_float) fail(LAQ_ERR_TYPE, "predicate constant is integer, column is float");
    if (p->kind < LAQ_PRED_LT || p->kind > LAQ_PRED_INSET) fail(LAQ_ERR_GENERIC, "unknown predicate kind");
    const int64_t sn = p->kind == LAQ_PRED_INSET ? p->set_len : 0;
    DevBuf<int64_t> dset(ctx, std::max<int64_t>(sn, 1));
    if (sn) {
      // the reference sorts the set at construction (predicate.hpp:67-79)
      std::vector<int64_t> s(sn);
      std::memcpy(s.data(), col_is_float ? static_cast<const void*>(p->fset) : static_cast<const void*>(p->iset),
                  sn * sizeof(int64_t));
      if (col_is_float) {
        std::vector<double> f(sn);
        std::memcpy(f.data(), s.data(), sn * 8);
        std::sort(f.begin(), f.end());
        std::memcpy(s.data(), f.data(), sn * 8);
      } else {
        std::sort(s.begin(), s.end());
      }
      LAQ_CUDA(cudaMemcpyAsync(dset.get(), s.data(), sn * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    }
    if (col_is_float)
      mask_kernel<double><<<blocks(ctx, n), kT, 0, ctx->stream>>>(static_cast<const double*>(d_col), n, p->kind, p->flo,
                                                                 p->fhi, reinterpret_cast<const double*>(dset.get()),
                                                                 sn, d_mask, and_into);
    else
      mask_kernel<int64_t><<<blocks(ctx, n), kT, 0, ctx->stream>>>(static_cast<const int64_t*>(d_col), n, p->kind,
                                                                  p->ilo, p->ihi, dset.get(), sn, d_mask, and_into);
    launched(ctx);
    sync(ctx);  // dset is freed on return
  });
}

int laq_mask_and(laq_ctx* ctx, const uint8_t* d_a, const uint8_t* d_b, int64_t n, uint8_t* d_out) {
  return guard(ctx, [&] {
    if (n <= 0) return;
    mask_and_kernel<<<blocks(ctx, n), kT, 0, ctx->stream>>>(d_a, d_b, n, d_out);
    launched(ctx);
  });
}

int laq_mask_indices(laq_ctx* ctx, const uint8_t* d_mask, int64_t n, int64_t* d_idx, int64_t* h_count) {
  return guard(ctx, [&] { *h_count = mask_positions(ctx, d_mask, n, d_idx); });
}

int laq_gather(laq_ctx* ctx, const void* d_src, int32_t src_kind, int64_t row_elems, const int64_t* d_idx, int64_t n,
               void* d_dst, int32_t out_kind) {
  return guard(ctx, [&] {
    if (src_kind < 0 || src_kind > 2 || out_kind < 1 || out_kind > 3 || (out_kind == 1 && src_kind == 2))
      fail(LAQ_ERR_SHAPE, "laq_gather: bad kinds");
    if (n <= 0 || row_elems <= 0) return;
    gather_kernel<<<blocks(ctx, n * row_elems), kT, 0, ctx->stream>>>(d_src, src_kind, row_elems, d_idx, n, d_dst,
                                                                       out_kind);
    launched(ctx);
  });
}

int laq_sum_f64(laq_ctx* ctx, const double* d_v, int64_t n, double* h_out) {
  return guard(ctx, [&] {
    *h_out = 0.0;
    if (n <= 0) return;
    // Integral values whose every partial sum stays below 2^53 add exactly in
    // any order: a parallel int64 reduction gives the sequential result.
    int* ne = reinterpret_cast<int*>(ctx->d_flags + 63);
    LAQ_CUDA(cudaMemsetAsync(ne, 0, sizeof(int), ctx->stream));
    const double limit = std::ldexp(1.0, 53) / static_cast<double>(n);
    integral_check_kernel<<<blocks(ctx, n), kT, 0, ctx->stream>>>(d_v, n, std::floor(limit), ne);
    launched(ctx);
    LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, ne, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    unsigned long long* acc = reinterpret_cast<unsigned long long*>(ctx->d_flags + 60);
    if (*reinterpret_cast<int*>(ctx->h_pinned) == 0) {
      LAQ_CUDA(cudaMemsetAsync(acc, 0, sizeof(unsigned long long), ctx->stream));
      sum_i64_kernel<<<blocks(ctx, n), kT, 0, ctx->stream>>>(d_v, n, acc);
      launched(ctx);
      LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, acc, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
      sync(ctx);
      *h_out = static_cast<double>(ctx->h_pinned[0]);
    } else {
      sum_seq_kernel<<<1, 32, 0, ctx->stream>>>(d_v, n, reinterpret_cast<double*>(acc));
      launched(ctx);
      LAQ_CUDA(cudaMemcpyAsync(h_out, acc, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      sync(ctx);
    }
  });
}

int laq_sort_rows(laq_ctx* ctx, const double* d_t, int64_t rows, int64_t cols, const int64_t* h_key_cols,
                  const int32_t* h_desc, int32_t n_keys, double* d_out) {
  return guard(ctx, [&] {
    for (int32_t k = 0; k < n_keys; ++k)
      if (h_key_cols[k] < 0 || h_key_cols[k] >= cols)
        fail(LAQ_ERR_INDEX, "sort_rows: key column " + std::to_string(h_key_cols[k]));
    if (rows <= 0 || cols <= 0) return;
    DevBuf<int64_t> perm(ctx, rows), perm2(ctx, rows);
    DevBuf<uint64_t> key(ctx, rows), skey(ctx, rows);
    iota_kernel<<<blocks(ctx, rows), kT, 0, ctx->stream>>>(perm.get(), rows);
    launched(ctx);
    // LSD over the keys (last key first), each pass a stable radix sort: the
    // final order is lexicographic with ties in the original row order.
    for (int32_t k = n_keys - 1; k >= 0; --k) {
      sort_key_kernel<<<blocks(ctx, rows), kT, 0, ctx->stream>>>(d_t, cols, h_key_cols[k], perm.get(), rows,
                                                                h_desc[k] != 0, key.get());
      launched(ctx);
      sort_pairs<uint64_t>(ctx, key.get(), skey.get(), perm.get(), perm2.get(), rows, 64);
      std::swap(perm, perm2);
    }
    gather_kernel<<<blocks(ctx, rows * cols), kT, 0, ctx->stream>>>(d_t, 2, cols, perm.get(), rows, d_out, 2);
    launched(ctx);
    sync(ctx);
  });
}

}  // extern "C"
