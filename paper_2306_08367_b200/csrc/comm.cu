// Row-sharded multi-GPU plumbing: one process per GPU, each
// holding a contiguous lineorder shard; the per-group int64 (count, sum)
// accumulators of a query are summed across ranks with ONE all-reduce
// (<= 2 x 280 int64 for SSB: latency-bound, ~10-20 us over NVLink 5), after
// which every rank emits the same rows.  The reference has no multi-process
// path (proj/README.md:115); this is the B200 build's.
//
// NCCL is loaded with dlopen("libnccl.so.2") on first use, so the library has
// no hard link dependency: in a PyTorch process that is the NCCL torch already
// loaded, in a plain C++ host the system one.  A host-side hook (any
// transport: gloo, MPI) can stand in for NCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace laq {
namespace {

struct Nccl {
  void* so = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!so) return;
    n.so = so;
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(so, "ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(so, "ncclCommInitRank"));
    n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(so, "ncclAllReduce"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(so, "ncclCommDestroy"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(so, "ncclGetErrorString"));
  });
  if (!n.so || !n.get_unique_id || !n.comm_init_rank || !n.all_reduce || !n.comm_destroy)
    fail(LAQ_ERR_UNSUPPORTED, "libnccl.so.2 could not be loaded");
  return n;
}

void check(const Nccl& n, ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(LAQ_ERR_CUDA, std::string(what) + ": " + (n.error_string ? n.error_string(r) : "nccl error"));
}

void detach(laq_ctx* ctx) {
  if (ctx->nccl) {
    const Nccl& n = nccl();
    n.comm_destroy(static_cast<ncclComm_t>(ctx->nccl));
    ctx->nccl = nullptr;
  }
  ctx->hook = nullptr;
  ctx->hook_user = nullptr;
  ctx->nranks = 1;
  ctx->rank = 0;
}

}  // namespace

void allreduce_i64(laq_ctx* ctx, int64_t* d_buf, int64_t count) {
  if (count <= 0) return;
  if (ctx->nccl) {
    const Nccl& n = nccl();
    check(n, n.all_reduce(d_buf, d_buf, static_cast<size_t>(count), ncclInt64, ncclSum,
                          static_cast<ncclComm_t>(ctx->nccl), ctx->stream),
          "ncclAllReduce");
  } else if (ctx->hook) {
    std::vector<int64_t> h(static_cast<size_t>(count));
    LAQ_CUDA(cudaMemcpyAsync(h.data(), d_buf, count * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    if (ctx->hook(h.data(), count, ctx->hook_user) != 0) fail(LAQ_ERR_GENERIC, "all-reduce hook failed");
    LAQ_CUDA(cudaMemcpyAsync(d_buf, h.data(), count * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    sync(ctx);
  }
}

}  // namespace laq

using namespace laq;

extern "C" {

int laq_nccl_unique_id(uint8_t h_id[128]) {
  return guard(nullptr, [&] {
    const Nccl& n = nccl();
    ncclUniqueId id;
    check(n, n.get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(h_id, id.internal, sizeof(id.internal));
  });
}

int laq_ctx_attach_nccl(laq_ctx* ctx, int32_t nranks, int32_t rank, const uint8_t h_id[128]) {
  return guard(ctx, [&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(LAQ_ERR_SHAPE, "bad rank / nranks");
    detach(ctx);
    if (nranks == 1) return;
    const Nccl& n = nccl();
    ncclUniqueId id;
    std::memcpy(id.internal, h_id, sizeof(id.internal));
    ncclComm_t comm = nullptr;
    // ncclCommInitRank binds the communicator to the calling thread's current
    // device: make that the context's device whatever the caller last set.
    LAQ_CUDA(cudaSetDevice(ctx->device));
    check(n, n.comm_init_rank(&comm, nranks, id, rank), "ncclCommInitRank");
    ctx->nccl = comm;
    ctx->nranks = nranks;
    ctx->rank = rank;
  });
}

int laq_ctx_set_allreduce_host(laq_ctx* ctx, int32_t nranks, int32_t rank, laq_allreduce_host_fn fn, void* user) {
  return guard(ctx, [&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(LAQ_ERR_SHAPE, "bad rank / nranks");
    detach(ctx);
    if (!fn) return;
    ctx->hook = fn;
    ctx->hook_user = user;
    ctx->nranks = nranks;
    ctx->rank = rank;
  });
}

int laq_ctx_comm_info(const laq_ctx* ctx, int32_t* h_nranks, int32_t* h_rank) {
  if (!ctx) return LAQ_ERR_GENERIC;
  *h_nranks = ctx->nranks;
  *h_rank = ctx->rank;
  return LAQ_OK;
}

int laq_allreduce_acc(laq_ctx* ctx, int64_t* d_acc, int64_t count) {
  return guard(ctx, [&] {
    if (count < 0) fail(LAQ_ERR_SHAPE, "negative count");
    allreduce_i64(ctx, d_acc, count);
  });
}

}  // extern "C"
