// Probe tables: the realisation of the one-hot join matrices.
//
// The reference joins fact rows to a dimension with
//   spmm(key_matrix(fks, D, RowsByDomain), key_matrix(pks, D, DomainByRows))
// (laqops.cpp:273-281).  With unique dimension keys each fact row has at most
// one nonzero in the product, at the dim row whose key equals the fact key.
// We never build the one-hot matrices: a probe table maps a key straight to
// its slot (the key's "domain position") and slot -> dim row, so one gather
// replaces key_matrix x key_matrix^T with zero wasted flops.
//
// Two layouts:
//  - DIRECT: slot = key - base for a key range not much larger than the row
//    count (every generated SSB key space: pk = iota).  One gather per probe.
//  - HASH:   open addressing (linear probing, power-of-two capacity >= 2x
//    rows) over arbitrary non-negative int64 keys.
#pragma once

#include "common.cuh"

namespace laq {

enum ProbeKind : int { PROBE_DIRECT = 0, PROBE_HASH = 1 };

struct ProbeView {
  int kind;
  int64_t base;         // DIRECT: smallest key
  int64_t size;         // DIRECT: key range; HASH: capacity (power of two)
  const int64_t* keys;  // HASH: key per slot (-1 = empty)
  const int32_t* rows;  // slot -> dim row (-1 = empty)

  // Slot of `key`, or -1.  Keys are non-negative (storage.cpp:54-56).
  __device__ __forceinline__ int64_t slot(int64_t key) const {
    if (kind == PROBE_DIRECT) {
      const uint64_t s = static_cast<uint64_t>(key - base);
      return s < static_cast<uint64_t>(size) ? static_cast<int64_t>(s) : -1;
    }
    const uint64_t mask = static_cast<uint64_t>(size) - 1;
    uint64_t h = static_cast<uint64_t>(key) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 29;
    for (uint64_t s = h & mask;; s = (s + 1) & mask) {
      const int64_t k = __ldg(keys + s);
      if (k == key) return static_cast<int64_t>(s);
      if (k < 0) return -1;
    }
  }
  __device__ __forceinline__ int32_t row(int64_t key) const {
    const int64_t s = slot(key);
    return s < 0 ? -1 : __ldg(rows + s);
  }
};

struct Probe {
  int kind = PROBE_DIRECT;
  int64_t base = 0, size = 0, n_rows = 0;
  DevMem<int64_t> keys;
  DevMem<int32_t> rows;
  DevMem<int32_t> row_slot;  // dim row -> slot (for per-query code tables)

  ProbeView view() const { return ProbeView{kind, base, size, keys.get(), rows.get()}; }
};

// Build a probe over n primary keys (int64 or int32 device array).
// Throws DomainError on a negative key and DuplicateKeyError (with `what`) on
// a duplicate (laqops.cpp:252-254).
// Views into a laq_probe (defined in probe.cu) for other kernels (ffn.cu).
int probe_links(const laq_probe* p);
ProbeView probe_view(const laq_probe* p, int j);

// pooled: the tables come from the context stream's pool (a probe that lives
// only inside one call; see DevMem).
void build_probe(laq_ctx* ctx, const int64_t* d_pk64, const int32_t* d_pk32, int64_t n, Probe& out,
                 const std::string& what, bool pooled = false);

// Sorted distinct values of a ++ b into out (count returned): a bitmap over
// [min, max] when the range is below 2^31, else radix sort + unique
// (keydomain.cu).  what != nullptr: negative values raise DomainError.
int64_t distinct_sorted(laq_ctx* ctx, const int64_t* a, int64_t na, const int64_t* b, int64_t nb, int64_t* out,
                        const char* what);

}  // namespace laq
