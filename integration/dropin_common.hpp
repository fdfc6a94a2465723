// Shared plumbing of the drop-in translation units (laq_dropin*.cpp): the
// process-wide C-ABI context, status -> laq::Error mapping, RAII device buffers.
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <string>
#include <vector>

#include "laq/error.hpp"
#include "laq/matrix.hpp"
#include "laq_b200.h"

namespace laq {
namespace dropin {

inline laq_ctx* ctx() {
  static laq_ctx* c = [] {
    laq_ctx* p = nullptr;
    const int rc = laq_ctx_create(0, &p);
    if (rc != LAQ_OK) throw Error("laq_b200: no usable sm_100 device (status " + std::to_string(rc) + ")");
    return p;
  }();
  return c;
}

[[noreturn]] inline void raise(int rc, const std::string& msg) {
  switch (rc) {
    case LAQ_ERR_INDEX: throw IndexError(msg);
    case LAQ_ERR_SHAPE: throw ShapeError(msg);
    case LAQ_ERR_FORMAT: throw FormatError(msg);
    case LAQ_ERR_NAME: throw NameError(msg);
    case LAQ_ERR_TYPE: throw TypeError(msg);
    case LAQ_ERR_MAPPING: throw MappingError(msg);
    case LAQ_ERR_DOMAIN: throw DomainError(msg);
    case LAQ_ERR_DUPLICATE_KEY: throw DuplicateKeyError(msg);
    case LAQ_ERR_TREE: throw TreeError(msg);
    case LAQ_ERR_MODEL: throw ModelError(msg);
    case LAQ_ERR_GEN: throw GenError(msg);
    case LAQ_ERR_CAPACITY: throw CapacityError(msg);
    default: throw Error(msg);
  }
}

inline void check(int rc) {
  if (rc != LAQ_OK) raise(rc, laq_ctx_last_error(ctx()));
}

// Device mirror of a host vector (freed on scope exit).  Allocated from the
// stream-ordered pool on the legacy stream, which the drop-in's context runs on
// (laq_ctx_create keeps freed blocks in the pool): a value-type call allocates
// and frees several buffers, and cudaMalloc/cudaFree synchronise the device.
template <class T>
struct Dev {
  T* p = nullptr;
  size_t n = 0;
  Dev() = default;
  explicit Dev(size_t count) : n(count) {
    ctx();
    if (n && cudaMallocAsync(reinterpret_cast<void**>(&p), n * sizeof(T), 0) != cudaSuccess)
      throw CapacityError("laq_b200: device allocation of " + std::to_string(n * sizeof(T)) + " bytes failed");
  }
  Dev(const T* h, size_t count) : Dev(count) { up(h, count); }
  explicit Dev(const std::vector<T>& v) : Dev(v.data(), v.size()) {}
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  Dev(Dev&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; }
  Dev& operator=(Dev&& o) noexcept {
    if (p) cudaFreeAsync(p, 0);
    p = o.p;
    n = o.n;
    o.p = nullptr;
    return *this;
  }
  ~Dev() {
    if (p) cudaFreeAsync(p, 0);
  }
  void up(const T* h, size_t m) {
    if (m && cudaMemcpy(p, h, m * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess) throw Error("laq_b200: H2D");
  }
  void down(T* h, size_t m) const {
    if (m && cudaMemcpy(h, p, m * sizeof(T), cudaMemcpyDeviceToHost) != cudaSuccess) throw Error("laq_b200: D2H");
  }
  std::vector<T> to_vector(size_t m) const {
    std::vector<T> v(m);
    down(v.data(), m);
    return v;
  }
};

inline std::string shape_str(index_t r, index_t c) { return std::to_string(r) + "x" + std::to_string(c); }

inline double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace dropin
}  // namespace laq
