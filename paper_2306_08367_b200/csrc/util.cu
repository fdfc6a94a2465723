// Context lifecycle, cost model and small device utilities (min/max, scans).
#include <cub/cub.cuh>

#include <algorithm>

#include <climits>
#include <cmath>

#include <cstring>
#include <type_traits>

#include "common.cuh"

namespace laq {

namespace {

template <class T>
__global__ void minmax_kernel(const T* __restrict__ d, int64_t n, unsigned long long* out_min_biased,
                              unsigned long long* out_max_biased) {
  // Bias by 2^63 so signed order == unsigned order for atomicMin/Max.
  int64_t mn = LLONG_MAX, mx = LLONG_MIN;
  auto take = [&](int64_t v) {
    mn = v < mn ? v : mn;
    mx = v > mx ? v : mx;
  };
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if ((reinterpret_cast<uintptr_t>(d) & 15) == 0) {
    // 16-byte loads, two per thread per step (64 B in flight per thread)
    constexpr int kPer = 16 / sizeof(T);
    using V = typename std::conditional<sizeof(T) == 8, longlong2, int4>::type;
    const V* v = reinterpret_cast<const V*>(d);
    const int64_t nv = n / kPer;
    int64_t i = tid;
    for (; i + nt < nv; i += 2 * nt) {
      const V a = __ldcs(v + i), b = __ldcs(v + i + nt);
      const T* pa = reinterpret_cast<const T*>(&a);
      const T* pb = reinterpret_cast<const T*>(&b);
#pragma unroll
      for (int k = 0; k < kPer; ++k) take(static_cast<int64_t>(pa[k])), take(static_cast<int64_t>(pb[k]));
    }
    for (; i < nv; i += nt) {
      const V a = __ldcs(v + i);
      const T* pa = reinterpret_cast<const T*>(&a);
#pragma unroll
      for (int k = 0; k < kPer; ++k) take(static_cast<int64_t>(pa[k]));
    }
    done = nv * kPer;
  }
  for (int64_t i = done + tid; i < n; i += nt) take(static_cast<int64_t>(d[i]));
  for (int o = 16; o; o >>= 1) {
    const int64_t a = __shfl_xor_sync(0xffffffffu, mn, o);
    const int64_t b = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out_min_biased, static_cast<unsigned long long>(mn) ^ 0x8000000000000000ull);
    atomicMax(out_max_biased, static_cast<unsigned long long>(mx) ^ 0x8000000000000000ull);
  }
}

template <class T>
void minmax_impl(laq_ctx* ctx, const T* d, int64_t n, int64_t* mn, int64_t* mx) {
  if (n == 0) {
    *mn = 0;
    *mx = -1;
    return;
  }
  unsigned long long* f = reinterpret_cast<unsigned long long*>(ctx->d_flags);
  unsigned long long init[2] = {~0ull, 0ull};
  LAQ_CUDA(cudaMemcpyAsync(f, init, sizeof init, cudaMemcpyHostToDevice, ctx->stream));
  minmax_kernel<T><<<grid_for(n, 256 * 16, ctx->sm_count * 8), 256, 0, ctx->stream>>>(d, n, f, f + 1);
  launched(ctx);
  LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, f, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  *mn = static_cast<int64_t>(static_cast<unsigned long long>(ctx->h_pinned[0]) ^ 0x8000000000000000ull);
  *mx = static_cast<int64_t>(static_cast<unsigned long long>(ctx->h_pinned[1]) ^ 0x8000000000000000ull);
}

}  // namespace

void minmax_i64(laq_ctx* ctx, const int64_t* d, int64_t n, int64_t* mn, int64_t* mx) { minmax_impl(ctx, d, n, mn, mx); }
void minmax_i32(laq_ctx* ctx, const int32_t* d, int64_t n, int64_t* mn, int64_t* mx) { minmax_impl(ctx, d, n, mn, mx); }

void exclusive_scan_i64(laq_ctx* ctx, const int64_t* d_in, int64_t* d_out, int64_t n, int64_t* h_total) {
  if (n == 0) {
    if (h_total) *h_total = 0;
    return;
  }
  size_t bytes = 0;
  LAQ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, d_in, d_out, n, ctx->stream));
  DevBuf<char> tmp(ctx, bytes);
  // Keep the last input element: d_in may alias d_out.
  int64_t* last_in = ctx->d_flags + 4;
  LAQ_CUDA(cudaMemcpyAsync(last_in, d_in + n - 1, sizeof(int64_t), cudaMemcpyDeviceToDevice, ctx->stream));
  LAQ_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, d_in, d_out, n, ctx->stream));
  ++ctx->launches;
  if (h_total) {
    LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, d_out + n - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned + 1, last_in, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    *h_total = ctx->h_pinned[0] + ctx->h_pinned[1];
  }
}

namespace {
__global__ void absmax_kernel(const double* __restrict__ x, int64_t n, unsigned long long* out) {
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(x[i]));
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(m)));
}
}  // namespace

double absmax_f64(laq_ctx* ctx, const double* d, int64_t n) {
  unsigned long long* f = reinterpret_cast<unsigned long long*>(ctx->d_flags + 58);
  LAQ_CUDA(cudaMemsetAsync(f, 0, sizeof(unsigned long long), ctx->stream));
  if (n > 0) {
    absmax_kernel<<<grid_for(n, 256, ctx->sm_count * 8), 256, 0, ctx->stream>>>(d, n, f);
    launched(ctx);
  }
  LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, f, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  double m;
  const int64_t bits = ctx->h_pinned[0];
  std::memcpy(&m, &bits, sizeof(m));
  return m;
}

}  // namespace laq

using namespace laq;

extern "C" {

#define LAQ_STR2(x) #x
#define LAQ_STR(x) LAQ_STR2(x)
const char* laq_version(void) { return "laq_b200 0.1 (sm_100a, cudart " LAQ_STR(CUDART_VERSION) ")"; }

int laq_ctx_create(int device, laq_ctx** out) {
  laq_ctx* ctx = new laq_ctx();
  ctx->device = device;
  const int rc = guard(ctx, [&] {
    int n = 0;
    LAQ_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) fail(LAQ_ERR_CUDA, "no such CUDA device");
    LAQ_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop{};
    LAQ_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) fail(LAQ_ERR_CUDA, std::string("built for sm_100a, device is ") + prop.name);
    ctx->sm_count = prop.multiProcessorCount;
    LAQ_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_pinned), 64 * sizeof(int64_t)));
    LAQ_CUDA(cudaMalloc(reinterpret_cast<void**>(&ctx->d_flags), 64 * sizeof(int64_t)));
    LAQ_CUDA(cudaMemset(ctx->d_flags, 0, 64 * sizeof(int64_t)));
    // Keep freed stream-ordered scratch in the pool instead of returning it to the driver.
    cudaMemPool_t pool;
    LAQ_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thresh = UINT64_MAX;
    LAQ_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
  });
  if (rc != LAQ_OK) {
    *out = nullptr;
    static thread_local std::string last;
    last = ctx->err;
    delete ctx;
    return rc;
  }
  *out = ctx;
  return LAQ_OK;
}

int laq_ctx_destroy(laq_ctx* ctx) {
  if (!ctx) return LAQ_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  laq_ctx_set_allreduce_host(ctx, 1, 0, nullptr, nullptr);  // releases an NCCL communicator
  if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
  if (ctx->d_flags) cudaFree(ctx->d_flags);
  delete ctx;
  return LAQ_OK;
}

int laq_ctx_set_stream(laq_ctx* ctx, void* s) {
  ctx->stream = static_cast<cudaStream_t>(s);
  return LAQ_OK;
}

int laq_ctx_synchronize(laq_ctx* ctx) {
  return guard(ctx, [&] { sync(ctx); });
}

const char* laq_ctx_last_error(const laq_ctx* ctx) { return ctx ? ctx->err.c_str() : "no context"; }
int64_t laq_ctx_launch_count(const laq_ctx* ctx) { return ctx ? ctx->launches : 0; }

// ---- cost model: fusion.cpp:181-224, verbatim formulas ----------------------
static int cost_check(int64_t i, int64_t k, int64_t l, int64_t p, const int64_t* dims, int32_t n) {
  if (i <= 0 || k <= 0 || l <= 0 || p <= 0) return LAQ_ERR_DOMAIN;
  if (n <= 0) return LAQ_ERR_DOMAIN;
  for (int32_t j = 0; j < n; ++j)
    if (dims[j] <= 0) return LAQ_ERR_DOMAIN;
  return LAQ_OK;
}

int laq_speedup_ratio_linear(int64_t i, int64_t k, int64_t l, const int64_t* dims, int32_t n, double* out) {
  // CostInputs::tree_features is validated too (fusion.cpp:189-197); linear callers pass k.
  const int rc = cost_check(i, k, l, k, dims, n);
  if (rc) return rc;
  double sum_r = 0;
  for (int32_t j = 0; j < n; ++j) sum_r += static_cast<double>(dims[j]);
  const double di = static_cast<double>(i), dk = static_cast<double>(k), dl = static_cast<double>(l);
  const double denom = di * dl * sum_r;
  if (denom == 0.0) return LAQ_ERR_DOMAIN;
  *out = ((di * dk + dk * dk / 3.0) * sum_r + di * dk * dl) / denom;
  return LAQ_OK;
}

int laq_speedup_ratio_tree(int64_t i, int64_t k, int64_t l, int64_t p, const int64_t* dims, int32_t n,
                           double* out) {
  const int rc = cost_check(i, k, l, p, dims, n);
  if (rc) return rc;
  double sum_r = 0;
  for (int32_t j = 0; j < n; ++j) sum_r += static_cast<double>(dims[j]);
  const double di = static_cast<double>(i), dk = static_cast<double>(k), dl = static_cast<double>(l);
  if (di * dl * sum_r == 0.0) return LAQ_ERR_DOMAIN;
  *out = dk / dl + dk * dk / (3.0 * di * dl) + dk * dk / (dl * sum_r) + dk / sum_r + dk / (dl * sum_r) +
         1.0 / sum_r;
  return LAQ_OK;
}

int laq_plan_linear_device(int64_t target_rows, int64_t k, int64_t l, const int64_t* dim_rows, int32_t n_dims,
                           double tensor_flops, double hbm_bytes_per_s, double* t_fused, double* t_nonfused,
                           int32_t* fused) {
  if (target_rows < 0 || k < 1 || l < 1 || n_dims < 1 || !dim_rows || tensor_flops <= 0 || hbm_bytes_per_s <= 0)
    return LAQ_ERR_DOMAIN;
  const double pt = tensor_flops * 0.85;   // tensor-pipe rate gemm_tc.cu reaches on long GEMMs
  const double bw = hbm_bytes_per_s * 0.76;  // gather + streaming mix
  const double ovh = 20e-6;                  // launch + pipeline fill per kernel
  const double F = static_cast<double>(target_rows);
  const double kp = static_cast<double>((k + 31) / 32 * 32);
  const double lp = static_cast<double>(std::max<int64_t>(16, (l + 15) / 16 * 16));
  const double dl = static_cast<double>(l), nd = static_cast<double>(n_dims);
  double R = 0, t_pre = 0;
  for (int32_t j = 0; j < n_dims; ++j) {
    if (dim_rows[j] < 0) return LAQ_ERR_DOMAIN;
    const double r = static_cast<double>(dim_rows[j]);
    R += r;
    t_pre += std::max(6.0 * r * kp * lp / pt, (r * kp * 4 + r * dl * 4) / bw);
  }
  // non-fused: one GEMM over the gathered rows (3 MMAs per product, fp16x2 split)
  const double t_nf = ovh + std::max(6.0 * F * kp * lp / pt, (F * 4 * nd + F * kp * 4 + F * dl * 4) / bw);
  // fused: P reads hit L2 while sum r_j l 4 B fits (~100 MB)
  const double gather_p = R * dl * 4 <= 100e6 ? 0.0 : F * dl * 4 * nd;
  const double t_f = (1 + nd) * ovh + t_pre + (F * 4 * nd + F * dl * 4 + gather_p) / bw;
  if (t_fused) *t_fused = t_f;
  if (t_nonfused) *t_nonfused = t_nf;
  if (fused) *fused = t_f < t_nf ? 1 : 0;
  return LAQ_OK;
}

int laq_decide_fusion(double ratio, double threshold, int32_t* out) {
  if (!std::isfinite(ratio)) return LAQ_ERR_DOMAIN;  // fusion.cpp:222
  *out = ratio > threshold ? 1 : 0;                   // strict, fusion.cpp:223
  return LAQ_OK;
}

}  // extern "C"
