// Shared host/device plumbing for the LAQ sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "laq_b200.h"

namespace laq {

// Host-side error carrying a laq_status; converted to a return code at the
// C-ABI boundary (guard()).
struct Err {
  int code;
  std::string msg;
};

[[noreturn]] inline void fail(int code, std::string msg) { throw Err{code, std::move(msg)}; }

#define LAQ_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      ::laq::fail(LAQ_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));     \
  } while (0)

constexpr int kNumSMs = 148;  // B200

}  // namespace laq

struct laq_ctx {
  int device = 0;
  int sm_count = laq::kNumSMs;
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t launches = 0;
  // Small pinned host staging for data-dependent sizes / flags.
  int64_t* h_pinned = nullptr;
  // Device flag words (error flags, counters) reused by synchronous calls.
  int64_t* d_flags = nullptr;
  // Row-sharded multi-GPU (comm.cu): an NCCL communicator over the
  // ranks that each hold one fact shard, or a host all-reduce hook supplied by
  // the caller (e.g. torch.distributed / MPI).  nranks == 1: single GPU.
  void* nccl = nullptr;  // ncclComm_t
  int32_t nranks = 1;
  int32_t rank = 0;
  laq_allreduce_host_fn hook = nullptr;
  void* hook_user = nullptr;
};

namespace laq {

// Run f() and translate exceptions into a status + ctx->err.
template <class F>
int guard(laq_ctx* ctx, F&& f) {
  try {
    if (ctx) LAQ_CUDA(cudaSetDevice(ctx->device));
    f();
    return LAQ_OK;
  } catch (const Err& e) {
    if (ctx) ctx->err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    return LAQ_ERR_GENERIC;
  }
}

// Launch bookkeeping: every kernel launch goes through this so the context can
// report how many of OUR kernels ran (bench.py "gpu_launches").
inline void launched(laq_ctx* ctx) {
  ++ctx->launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(LAQ_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
}

inline void sync(laq_ctx* ctx) { LAQ_CUDA(cudaStreamSynchronize(ctx->stream)); }

// Stream-ordered device scratch that frees itself (cudaMallocAsync pool).
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(laq_ctx* ctx, size_t count) : n(count), s(ctx->stream) {
    if (count) LAQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), s));
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    reset();
    p = o.p; n = o.n; s = o.s; o.p = nullptr;
    return *this;
  }
  ~DevBuf() { reset(); }
  void reset() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
  }
  T* get() const { return p; }
};

// Persistent device allocation (plans, probe tables): plain cudaMalloc.  The
// (count, ctx) form takes the memory from the context stream's pool instead
// and frees it stream-ordered: for per-call temporaries (a probe built and
// dropped inside one C-ABI call) that would otherwise pay a synchronising
// cudaMalloc/cudaFree each call.
template <class T>
struct DevMem {
  T* p = nullptr;
  size_t n = 0;
  bool pooled = false;
  cudaStream_t s = nullptr;
  DevMem() = default;
  explicit DevMem(size_t count) : n(count) {
    if (count) LAQ_CUDA(cudaMalloc(reinterpret_cast<void**>(&p), count * sizeof(T)));
  }
  DevMem(size_t count, const laq_ctx* ctx) : n(count), pooled(true), s(ctx->stream) {
    if (count) LAQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), s));
  }
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
  DevMem(DevMem&& o) noexcept : p(o.p), n(o.n), pooled(o.pooled), s(o.s) { o.p = nullptr; }
  DevMem& operator=(DevMem&& o) noexcept {
    release();
    p = o.p; n = o.n; pooled = o.pooled; s = o.s; o.p = nullptr;
    return *this;
  }
  ~DevMem() { release(); }
  void release() {
    if (p) {
      if (pooled) cudaFreeAsync(p, s);
      else cudaFree(p);
    }
    p = nullptr;
  }
  T* get() const { return p; }
};

template <class T>
DevMem<T> dev_mem(int64_t count, const laq_ctx* ctx, bool pooled) {
  return pooled ? DevMem<T>(static_cast<size_t>(count), ctx) : DevMem<T>(static_cast<size_t>(count));
}

// Bits needed for every value in [0, max_val] (>= 1; 64 for a negative max_val):
// the end_bit of a radix sort over keys known to lie in that range.
inline int bits_for(int64_t max_val) {
  if (max_val < 0) return 64;
  int b = 1;
  while (b < 63 && (max_val >> b) != 0) ++b;
  return b;
}

inline int grid_for(int64_t n, int per_block, int max_blocks) {
  int64_t b = (n + per_block - 1) / per_block;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return static_cast<int>(b);
}

// ---- shared helpers implemented in util.cu -----------------------------
// min/max of an int64 or int32 array (device reduce, synchronises).
void minmax_i64(laq_ctx* ctx, const int64_t* d, int64_t n, int64_t* mn, int64_t* mx);
void minmax_i32(laq_ctx* ctx, const int32_t* d, int64_t n, int64_t* mn, int64_t* mx);
// max |x| over a device fp64 array (synchronises); 0 for n == 0.
double absmax_f64(laq_ctx* ctx, const double* d, int64_t n);
// Exclusive scan of int64 counts (in place allowed); returns total (synchronises
// only when h_total != nullptr).
void exclusive_scan_i64(laq_ctx* ctx, const int64_t* d_in, int64_t* d_out, int64_t n, int64_t* h_total);
// Sum d_buf (count int64, on ctx->stream) across the context's ranks: NCCL when
// a communicator is attached, else the host hook, else nothing (comm.cu).
void allreduce_i64(laq_ctx* ctx, int64_t* d_buf, int64_t count);
inline bool sharded(const laq_ctx* ctx) { return ctx->nranks > 1 || ctx->hook != nullptr; }

}  // namespace laq
