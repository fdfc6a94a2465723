// K1 domain_build and the general (many-to-many) join-MM.
//
// build_key_domain (laqops.cpp:142-155) is "sorted distinct union".  For key
// ranges up to 2^31 we never sort: a bitmap over [min, max] (atomicOr), a
// per-word popcount, an exclusive scan of the counts, and an emit pass that
// writes each set bit's key at  offset[word] + popc(word & lower bits)  --
// ascending order for free, and that same rank is KeyDomain::position.
// Wider key spaces fall back to an on-device radix sort + unique.
//
// mm_join (laqops.cpp:222-231) = spmm(key_matrix(R), key_matrix(S)^T): S is
// bucketed by key with a stable radix sort (the DomainByRows CSR of S:
// buckets ascending, rows ascending within a bucket), each R row probes its
// bucket, a scan of bucket sizes gives output offsets, and the pairs are
// written in canonical (r asc, s asc) order.
#include <cub/cub.cuh>

#include <algorithm>

#include "probe.cuh"

namespace laq {
namespace {

__global__ void bitmap_set(const int64_t* __restrict__ k, int64_t n, int64_t base, unsigned* bits) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = k[i] - base;
    atomicOr(bits + (o >> 5), 1u << (o & 31));
  }
}

// Key ranges whose bitmap fits one CTA's shared memory (<= kSmemBitmapWords
// words, ~1.6M keys): every CTA sets bits in its own shared copy (shared
// atomics, no L2 contention -- 60M keys over a 1M range put ~1,900 global
// atomics on every word), then ORs its non-zero words into the global bitmap.
// Both key arrays in one launch; 16-byte streaming loads of two keys.
constexpr int kBitmapThreads = 1024;
constexpr int64_t kSmemBitmapWords = 50 * 1024;

__device__ __forceinline__ void smem_set_bit(unsigned* sb, int64_t key, int64_t base) {
  // Skip the atomic when the bit is already set (a plain shared load): with
  // few distinct keys every CTA's atomics would otherwise serialise on a
  // handful of words.  A stale read only costs a redundant atomic.
  const uint32_t o = static_cast<uint32_t>(key - base);
  const unsigned bit = 1u << (o & 31);
  if (!(*reinterpret_cast<volatile unsigned*>(sb + (o >> 5)) & bit)) atomicOr(sb + (o >> 5), bit);
}

__device__ __forceinline__ void smem_set_keys(unsigned* sb, const int64_t* __restrict__ k, int64_t n, int64_t base) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  int64_t head = 0;
  if (reinterpret_cast<uintptr_t>(k) & 15) {  // align the vector loop to 16 bytes
    head = 1;
    if (tid == 0 && n > 0) smem_set_bit(sb, k[0], base);
  }
  const int64_t pairs = (n - head) / 2;
  const longlong2* v = reinterpret_cast<const longlong2*>(k + head);
  for (int64_t i = tid; i < pairs; i += nt) {
    const longlong2 x = __ldcs(v + i);
    smem_set_bit(sb, x.x, base);
    smem_set_bit(sb, x.y, base);
  }
  if (tid == 0 && head + 2 * pairs < n) smem_set_bit(sb, k[n - 1], base);
}

__global__ void __launch_bounds__(kBitmapThreads) bitmap_set_smem(const int64_t* __restrict__ a, int64_t na,
                                                                  const int64_t* __restrict__ b, int64_t nb,
                                                                  int64_t base, int64_t words, unsigned* bits) {
  extern __shared__ unsigned sb[];
  for (int64_t w = threadIdx.x; w < words; w += blockDim.x) sb[w] = 0;
  __syncthreads();
  smem_set_keys(sb, a, na, base);
  smem_set_keys(sb, b, nb, base);
  __syncthreads();
  for (int64_t w = threadIdx.x; w < words; w += blockDim.x)
    if (const unsigned x = sb[w]) atomicOr(bits + w, x);
}

__global__ void bitmap_popc(const unsigned* __restrict__ bits, int64_t words, int64_t* cnt) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x)
    cnt[w] = __popc(bits[w]);
}

__global__ void bitmap_emit(const unsigned* __restrict__ bits, const int64_t* __restrict__ off, int64_t words,
                            int64_t base, int64_t* out) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x) {
    unsigned b = bits[w];
    int64_t o = off[w];
    while (b) {
      const int bit = __ffs(b) - 1;
      out[o++] = base + w * 32 + bit;
      b &= b - 1;
    }
  }
}

// a ++ b, minus `base` (the minimum): the keys become offsets in [0, range]
// so the radix sort only needs the range's significant bits.
__global__ void copy_i64(const int64_t* __restrict__ a, int64_t na, const int64_t* __restrict__ b, int64_t nb,
                         int64_t base, int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < na + nb; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = static_cast<int64_t>(static_cast<uint64_t>(i < na ? a[i] : b[i - na]) - static_cast<uint64_t>(base));
}

__global__ void add_base(int64_t* __restrict__ v, const int64_t* __restrict__ n, int64_t base) {
  const int64_t m = *n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = static_cast<int64_t>(static_cast<uint64_t>(v[i]) + static_cast<uint64_t>(base));
}

}  // namespace

// Sorted distinct keys of the concatenation a ++ b into out; returns count.
// what != nullptr: negative keys raise DomainError (join keys); nullptr: any
// int64 values (group-by columns).
int64_t distinct_sorted(laq_ctx* ctx, const int64_t* a, int64_t na, const int64_t* b, int64_t nb, int64_t* out,
                        const char* what) {
  const int64_t n = na + nb;
  if (n == 0) return 0;
  int64_t mn = INT64_MAX, mx = INT64_MIN, t0, t1;
  if (na) { minmax_i64(ctx, a, na, &t0, &t1); mn = std::min(mn, t0); mx = std::max(mx, t1); }
  if (nb) { minmax_i64(ctx, b, nb, &t0, &t1); mn = std::min(mn, t0); mx = std::max(mx, t1); }
  if (what && mn < 0) fail(LAQ_ERR_DOMAIN, std::string(what) + std::to_string(mn));
  const bool narrow = static_cast<uint64_t>(mx) - static_cast<uint64_t>(mn) < (uint64_t{1} << 31);
  const int64_t range = narrow ? mx - mn + 1 : 0;
  if (narrow) {
    const int64_t words = (range + 31) / 32;
    DevBuf<unsigned> bits(ctx, words);
    DevBuf<int64_t> cnt(ctx, words);
    LAQ_CUDA(cudaMemsetAsync(bits.get(), 0, words * sizeof(unsigned), ctx->stream));
    const int g = ctx->sm_count * 8;
    if (words <= kSmemBitmapWords && n >= 64 * words) {
      // Dense keys (many keys per bitmap word): per-CTA shared-memory bitmaps.
      const size_t smem = static_cast<size_t>(words) * sizeof(unsigned);
      LAQ_CUDA(cudaFuncSetAttribute(bitmap_set_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSmemBitmapWords * sizeof(unsigned))));
      const int blocks = static_cast<int>(std::min<int64_t>(ctx->sm_count, (n + 2 * kBitmapThreads - 1) / (2 * kBitmapThreads)));
      bitmap_set_smem<<<blocks, kBitmapThreads, smem, ctx->stream>>>(a, na, b, nb, mn, words, bits.get());
      launched(ctx);
    } else {
      if (na) { bitmap_set<<<grid_for(na, 256, g), 256, 0, ctx->stream>>>(a, na, mn, bits.get()); launched(ctx); }
      if (nb) { bitmap_set<<<grid_for(nb, 256, g), 256, 0, ctx->stream>>>(b, nb, mn, bits.get()); launched(ctx); }
    }
    bitmap_popc<<<grid_for(words, 256, g), 256, 0, ctx->stream>>>(bits.get(), words, cnt.get());
    launched(ctx);
    int64_t total = 0;
    exclusive_scan_i64(ctx, cnt.get(), cnt.get(), words, &total);
    bitmap_emit<<<grid_for(words, 256, g), 256, 0, ctx->stream>>>(bits.get(), cnt.get(), words, mn, out);
    launched(ctx);
    return total;
  }
  // Wide key space: radix sort + unique.  When the range fits 63 bits the keys
  // are sorted as offsets from the minimum over the range's bits only (2^40
  // keys: 5 onesweep passes instead of 8), and the minimum is added back to the
  // distinct offsets.
  const uint64_t urange = static_cast<uint64_t>(mx) - static_cast<uint64_t>(mn);
  const bool offs = urange < (uint64_t{1} << 63);
  const int64_t base = offs ? mn : 0;
  const int bits = offs ? bits_for(static_cast<int64_t>(urange)) : 64;
  DevBuf<int64_t> cat(ctx, n), sorted(ctx, n);
  copy_i64<<<grid_for(n, 256, ctx->sm_count * 8), 256, 0, ctx->stream>>>(a, na, b, nb, base, cat.get());
  launched(ctx);
  size_t bytes = 0;
  LAQ_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, cat.get(), sorted.get(), n, 0, bits, ctx->stream));
  DevBuf<char> tmp(ctx, bytes);
  LAQ_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(), bytes, cat.get(), sorted.get(), n, 0, bits, ctx->stream));
  ++ctx->launches;
  int64_t* d_num = ctx->d_flags + 40;
  size_t b2 = 0;
  LAQ_CUDA(cub::DeviceSelect::Unique(nullptr, b2, sorted.get(), out, d_num, n, ctx->stream));
  DevBuf<char> tmp2(ctx, b2);
  LAQ_CUDA(cub::DeviceSelect::Unique(tmp2.get(), b2, sorted.get(), out, d_num, n, ctx->stream));
  ++ctx->launches;
  if (base != 0) {
    add_base<<<grid_for(n, 256, ctx->sm_count * 8), 256, 0, ctx->stream>>>(out, d_num, base);
    launched(ctx);
  }
  LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, d_num, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  return ctx->h_pinned[0];
}

namespace {

// Keys -> domain positions.  A contiguous domain (its sorted distinct keys are
// exactly base .. base + d - 1, e.g. dense surrogate keys) needs no table:
// position = key - base, so the kernel streams 8 B in and 8 B out per key with
// 16-byte loads/stores (CONTIG).  Otherwise each key gathers its slot from the
// probe table (L2-resident; one key per thread per step measured fastest --
// four independent gathers per thread were 1.2-1.4x slower, bound by L2
// sector throughput).  One flag write per warp that saw a miss.
template <bool CONTIG>
__global__ void positions_kernel(const int64_t* __restrict__ keys, int64_t n, const ProbeView pv, int64_t* pos,
                                 int* missing) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  bool miss = false;
  auto contig = [&](int64_t key) -> int64_t {
    const uint64_t s = static_cast<uint64_t>(key - pv.base);
    const bool in = s < static_cast<uint64_t>(pv.size);
    miss = miss || !in;
    return in ? static_cast<int64_t>(s) : -1;
  };
  int64_t done = 0;
  if constexpr (CONTIG) {
    if (((reinterpret_cast<uintptr_t>(keys) | reinterpret_cast<uintptr_t>(pos)) & 15) == 0) {
      const int64_t pairs = n / 2;
      const longlong2* kv = reinterpret_cast<const longlong2*>(keys);
      longlong2* pv2 = reinterpret_cast<longlong2*>(pos);
      for (int64_t i = tid; i < pairs; i += nt) {
        const longlong2 x = __ldcs(kv + i);
        longlong2 p;
        p.x = contig(x.x);
        p.y = contig(x.y);
        __stcs(pv2 + i, p);
      }
      done = 2 * pairs;
    }
    for (int64_t i = done + tid; i < n; i += nt) pos[i] = contig(keys[i]);
  } else {
    for (int64_t i = tid; i < n; i += nt) {
      const int64_t k = keys[i];
      const int32_t r = k < 0 ? -1 : pv.row(k);
      miss = miss || r < 0;
      pos[i] = r;
    }
  }
  if (__any_sync(0xffffffffu, miss) && (threadIdx.x & 31) == 0) atomicOr(missing, 1);
}

// Positions of keys in a sorted distinct domain (DomainError if absent).
void positions(laq_ctx* ctx, const int64_t* keys, int64_t n, const int64_t* domain, int64_t d, int64_t* pos,
               Probe& probe_out) {
  build_probe(ctx, domain, nullptr, d, probe_out, "key domain has duplicate keys", /*pooled=*/true);
  int* missing = reinterpret_cast<int*>(ctx->d_flags + 41);
  LAQ_CUDA(cudaMemsetAsync(missing, 0, sizeof(int), ctx->stream));
  if (n) {
    // build_probe rejected duplicates, so a DIRECT probe whose key range equals
    // the domain size holds every key of [base, base + d): a contiguous domain.
    if (probe_out.kind == PROBE_DIRECT && probe_out.size == d)
      positions_kernel<true><<<grid_for(n, 256 * 2, ctx->sm_count * 8), 256, 0, ctx->stream>>>(
          keys, n, probe_out.view(), pos, missing);
    else
      positions_kernel<false><<<grid_for(n, 256, ctx->sm_count * 8), 256, 0, ctx->stream>>>(
          keys, n, probe_out.view(), pos, missing);
    launched(ctx);
  }
  LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, missing, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  if (*reinterpret_cast<int*>(ctx->h_pinned)) fail(LAQ_ERR_DOMAIN, "key not in domain");
}

__global__ void iota_i64(int64_t* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i;
}

// CSR row pointers from the sorted positions: row_ptr[p] = the first index
// whose position is >= p.  Thread i owns the positions in (spos[i-1], spos[i]]
// (with spos[-1] = -1 and spos[m] = d), so every row_ptr entry is written once
// and empty positions get their successor's start -- no atomics, no scan.
__global__ void row_ptr_from_sorted(const int64_t* __restrict__ spos, int64_t m, int64_t d, int64_t* row_ptr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= m; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = i == 0 ? -1 : spos[i - 1];
    const int64_t b = i == m ? d : spos[i];
    for (int64_t p = a + 1; p <= b; ++p) row_ptr[p] = i;
  }
}

// The same row pointers by one lower-bound binary search per position: for
// domains much smaller than the entry count (d <= m / 16: d log m reads
// instead of m), and free of the boundary form's serial loop over a long run
// of empty positions.
__global__ void row_ptr_by_search(const int64_t* __restrict__ spos, int64_t m, int64_t d, int64_t* row_ptr) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p <= d; p += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(spos + mid) < p) lo = mid + 1; else hi = mid;
    }
    row_ptr[p] = lo;
  }
}

__global__ void nonzero_flags(const double* __restrict__ v, int64_t n, char* flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = v[i] != 0.0;
}

__global__ void gather_values(const double* __restrict__ v, const int64_t* __restrict__ idx, int64_t m, double* out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = v ? v[idx[t]] : 1.0;
}

// mm_join: per R row, bucket lookup; write pairs.
__global__ void mm_count(const int64_t* __restrict__ r, int64_t nr, const ProbeView pv, const int64_t* __restrict__ run_off,
                         int64_t* cnt, int64_t* run_of_r) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nr; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = pv.row(r[i]);
    run_of_r[i] = u;
    cnt[i] = u < 0 ? 0 : run_off[u + 1] - run_off[u];
  }
}

__global__ void mm_write(int64_t nr, const int64_t* __restrict__ run_of_r, const int64_t* __restrict__ run_off,
                         const int64_t* __restrict__ s_sorted_idx, const int64_t* __restrict__ out_off, int64_t* out_r,
                         int64_t* out_s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nr; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = run_of_r[i];
    if (u < 0) continue;
    int64_t o = out_off[i];
    for (int64_t t = run_off[u]; t < run_off[u + 1]; ++t, ++o) {
      out_r[o] = i;
      out_s[o] = s_sorted_idx[t];
    }
  }
}

}  // namespace

// Shared with groupby.cu: S rows bucketed by key (stable), distinct keys probe.
struct Buckets {
  DevBuf<int64_t> sorted_keys, sorted_idx, uniq, run_off;
  int64_t n_uniq = 0;
  Probe probe;  // over uniq keys: row = run index
};

// keys are non-negative and <= max_key (max_key < 0: unknown, sort all 64 bits).
void bucket_by_key(laq_ctx* ctx, const int64_t* keys, int64_t n, Buckets& b, int64_t max_key) {
  b.sorted_keys = DevBuf<int64_t>(ctx, std::max<int64_t>(n, 1));
  b.sorted_idx = DevBuf<int64_t>(ctx, std::max<int64_t>(n, 1));
  b.uniq = DevBuf<int64_t>(ctx, std::max<int64_t>(n, 1));
  b.run_off = DevBuf<int64_t>(ctx, n + 1);
  if (n == 0) {
    LAQ_CUDA(cudaMemsetAsync(b.run_off.get(), 0, sizeof(int64_t), ctx->stream));
    b.n_uniq = 0;
    build_probe(ctx, b.uniq.get(), nullptr, 0, b.probe, "", /*pooled=*/true);
    return;
  }
  DevBuf<int64_t> iota(ctx, n);
  iota_i64<<<grid_for(n, 256, ctx->sm_count * 8), 256, 0, ctx->stream>>>(iota.get(), n);
  launched(ctx);
  size_t bytes = 0;
  const int bits = max_key < 0 ? 64 : bits_for(max_key);
  LAQ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, b.sorted_keys.get(), iota.get(), b.sorted_idx.get(), n,
                                           0, bits, ctx->stream));
  DevBuf<char> tmp(ctx, bytes);
  LAQ_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, keys, b.sorted_keys.get(), iota.get(), b.sorted_idx.get(),
                                           n, 0, bits, ctx->stream));
  ++ctx->launches;
  DevBuf<int64_t> counts(ctx, n);
  int64_t* d_runs = ctx->d_flags + 42;
  size_t b2 = 0;
  LAQ_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, b2, b.sorted_keys.get(), b.uniq.get(), counts.get(), d_runs, n,
                                              ctx->stream));
  DevBuf<char> tmp2(ctx, b2);
  LAQ_CUDA(cub::DeviceRunLengthEncode::Encode(tmp2.get(), b2, b.sorted_keys.get(), b.uniq.get(), counts.get(), d_runs,
                                              n, ctx->stream));
  ++ctx->launches;
  LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, d_runs, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  b.n_uniq = ctx->h_pinned[0];
  int64_t total = 0;
  exclusive_scan_i64(ctx, counts.get(), b.run_off.get(), b.n_uniq, &total);
  ctx->h_pinned[8] = total;
  LAQ_CUDA(cudaMemcpyAsync(b.run_off.get() + b.n_uniq, &ctx->h_pinned[8], sizeof(int64_t), cudaMemcpyHostToDevice,
                           ctx->stream));
  sync(ctx);
  build_probe(ctx, b.uniq.get(), nullptr, b.n_uniq, b.probe, "", /*pooled=*/true);
}

}  // namespace laq

using namespace laq;

extern "C" {

int laq_build_key_domain(laq_ctx* ctx, const int64_t* r, int64_t nr, const int64_t* s, int64_t ns, int64_t* out,
                         int64_t* h_size) {
  return guard(ctx, [&] { *h_size = distinct_sorted(ctx, r, nr, s, ns, out, "negative join key "); });
}

int laq_update_key_domain(laq_ctx* ctx, const int64_t* dom, int64_t d, const int64_t* nk, int64_t nn, int64_t* out,
                          int64_t* h_size) {
  // Merging into a sorted distinct domain == the distinct union (laqops.cpp:157-171).
  return guard(ctx, [&] { *h_size = distinct_sorted(ctx, dom, d, nk, nn, out, "negative join key "); });
}

int laq_key_positions(laq_ctx* ctx, const int64_t* keys, int64_t n, const int64_t* domain, int64_t d, int64_t* pos) {
  return guard(ctx, [&] {
    Probe p;
    positions(ctx, keys, n, domain, d, pos, p);
  });
}

int laq_key_matrix_dbr(laq_ctx* ctx, const int64_t* keys, int64_t n, const int64_t* domain, int64_t d,
                       const double* values, int64_t* row_ptr, int64_t* col_idx, double* out_values, int64_t* h_nnz) {
  return guard(ctx, [&] {
    // Counting sort by domain position; rows ascending within a position
    // (laqops.cpp:196-218).  Entries with value exactly 0.0 are validated but not stored.
    DevBuf<int64_t> pos(ctx, std::max<int64_t>(n, 1));
    Probe p;
    positions(ctx, keys, n, domain, d, pos.get(), p);
    // Keep-mask compaction (stable) for valued matrices.
    DevBuf<int64_t> kpos(ctx, std::max<int64_t>(n, 1)), kidx(ctx, std::max<int64_t>(n, 1));
    int64_t m = n;
    DevBuf<int64_t> iota(ctx, std::max<int64_t>(n, 1));
    if (n) {
      iota_i64<<<grid_for(n, 256, ctx->sm_count * 8), 256, 0, ctx->stream>>>(iota.get(), n);
      launched(ctx);
    }
    if (values && n) {
      DevBuf<char> flags(ctx, n);
      nonzero_flags<<<grid_for(n, 256, ctx->sm_count * 8), 256, 0, ctx->stream>>>(values, n, flags.get());
      launched(ctx);
      int64_t* d_cnt = ctx->d_flags + 43;
      size_t b = 0;
      LAQ_CUDA(cub::DeviceSelect::Flagged(nullptr, b, pos.get(), flags.get(), kpos.get(), d_cnt, n, ctx->stream));
      DevBuf<char> t(ctx, b);
      LAQ_CUDA(cub::DeviceSelect::Flagged(t.get(), b, pos.get(), flags.get(), kpos.get(), d_cnt, n, ctx->stream));
      LAQ_CUDA(cub::DeviceSelect::Flagged(t.get(), b, iota.get(), flags.get(), kidx.get(), d_cnt, n, ctx->stream));
      ctx->launches += 2;
      LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, d_cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
      sync(ctx);
      m = ctx->h_pinned[0];
    } else if (n) {
      LAQ_CUDA(cudaMemcpyAsync(kpos.get(), pos.get(), n * sizeof(int64_t), cudaMemcpyDeviceToDevice, ctx->stream));
      LAQ_CUDA(cudaMemcpyAsync(kidx.get(), iota.get(), n * sizeof(int64_t), cudaMemcpyDeviceToDevice, ctx->stream));
    }
    // Stable sort of (pos, row) by pos -> col_idx; histogram + scan -> row_ptr.
    DevBuf<int64_t> spos(ctx, std::max<int64_t>(m, 1));
    if (m) {
      size_t bytes = 0;
      const int bits = bits_for(d - 1);  // positions lie in [0, d): sort only their significant bits
      LAQ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kpos.get(), spos.get(), kidx.get(), col_idx, m, 0, bits,
                                               ctx->stream));
      DevBuf<char> tmp(ctx, bytes);
      LAQ_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, kpos.get(), spos.get(), kidx.get(), col_idx, m, 0, bits,
                                               ctx->stream));
      ++ctx->launches;
    }
    if (d > m / 16)  // positions comparable in number to the entries: one pass over the entries
      row_ptr_from_sorted<<<grid_for(m + 1, 256, ctx->sm_count * 8), 256, 0, ctx->stream>>>(spos.get(), m, d, row_ptr);
    else
      row_ptr_by_search<<<grid_for(d + 1, 256, ctx->sm_count * 8), 256, 0, ctx->stream>>>(spos.get(), m, d, row_ptr);
    launched(ctx);
    if (out_values && m) {
      gather_values<<<grid_for(m, 256, ctx->sm_count * 8), 256, 0, ctx->stream>>>(values, col_idx, m, out_values);
      launched(ctx);
    }
    sync(ctx);
    *h_nnz = m;
  });
}

int laq_mm_join(laq_ctx* ctx, const int64_t* r, int64_t nr, const int64_t* s, int64_t ns, int64_t* out_r,
                int64_t* out_s, int64_t capacity, int64_t* h_nnz) {
  return guard(ctx, [&] {
    // Domain validation as build_key_domain(keys_r, keys_s) (negative keys).
    int64_t mn, mx = -1;
    if (nr) { minmax_i64(ctx, r, nr, &mn, &mx); if (mn < 0) fail(LAQ_ERR_DOMAIN, "negative join key " + std::to_string(mn)); }
    mx = -1;
    if (ns) { minmax_i64(ctx, s, ns, &mn, &mx); if (mn < 0) fail(LAQ_ERR_DOMAIN, "negative join key " + std::to_string(mn)); }
    Buckets b;
    bucket_by_key(ctx, s, ns, b, mx);  // S keys in [0, mx]
    DevBuf<int64_t> cnt(ctx, std::max<int64_t>(nr, 1)), run_of_r(ctx, std::max<int64_t>(nr, 1)),
        off(ctx, std::max<int64_t>(nr, 1));
    int64_t total = 0;
    if (nr) {
      mm_count<<<grid_for(nr, 256, ctx->sm_count * 8), 256, 0, ctx->stream>>>(r, nr, b.probe.view(), b.run_off.get(),
                                                                              cnt.get(), run_of_r.get());
      launched(ctx);
      exclusive_scan_i64(ctx, cnt.get(), off.get(), nr, &total);
    }
    *h_nnz = total;
    if (total > capacity) fail(LAQ_ERR_CAPACITY, "mm_join: output capacity " + std::to_string(capacity) + " < " + std::to_string(total));
    if (nr && total) {
      mm_write<<<grid_for(nr, 256, ctx->sm_count * 8), 256, 0, ctx->stream>>>(nr, run_of_r.get(), b.run_off.get(),
                                                                              b.sorted_idx.get(), off.get(), out_r, out_s);
      launched(ctx);
      sync(ctx);
    }
  });
}

}  // extern "C"
