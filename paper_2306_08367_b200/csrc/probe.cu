// K2 star_probe + K3 fused_gather_sum: the star join evaluated as probes into
// one-hot key tables (probe.cuh), stable survivor compaction with a
// single-pass decoupled look-back scan, and the fused join+predict
//   Y[m] = ((P_0[row_0(m)] + P_1[row_1(m)]) + ...)
// for the m-th surviving fact row (fusion.cpp:64-77 association order; the
// one-hot gathers are exact, so the result is bit-identical to the reference).
//
// HBM traffic per fact row: 4*J bytes of int32 keys in, 8*l bytes of fp64
// predictions out (partials P_j are L2/L1 resident: r_j*l*8 bytes each).
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>

#include "predict_slot.cuh"
#include "probe.cuh"

namespace laq {

namespace {

constexpr int kMaxLinks = 8;
constexpr int kBlock = 256;
constexpr int kItems = 8;               // consecutive fact rows per thread
constexpr int kTile = kBlock * kItems;  // 2048 rows per tile

// ---------------------------------------------------------------------------
// probe construction
// ---------------------------------------------------------------------------

template <class K>
__global__ void direct_insert(const K* __restrict__ pk, int64_t n, int64_t base, int32_t* rows, int32_t* row_slot,
                              int* dup) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = static_cast<int64_t>(pk[r]) - base;
    const int32_t prev = atomicCAS(rows + s, -1, static_cast<int32_t>(r));
    if (prev != -1) atomicOr(dup, 1);
    row_slot[r] = static_cast<int32_t>(s);
  }
}

template <class K>
__global__ void hash_insert(const K* __restrict__ pk, int64_t n, int64_t cap, unsigned long long* keys, int32_t* rows,
                            int32_t* row_slot, int* dup) {
  const uint64_t mask = static_cast<uint64_t>(cap) - 1;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t key = static_cast<int64_t>(pk[r]);
    uint64_t h = static_cast<uint64_t>(key) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 29;
    for (uint64_t s = h & mask;; s = (s + 1) & mask) {
      const unsigned long long prev = atomicCAS(keys + s, ~0ull, static_cast<unsigned long long>(key));
      if (prev == ~0ull) {
        rows[s] = static_cast<int32_t>(r);
        row_slot[r] = static_cast<int32_t>(s);
        break;
      }
      if (prev == static_cast<unsigned long long>(key)) {
        atomicOr(dup, 1);
        row_slot[r] = static_cast<int32_t>(s);
        break;
      }
    }
  }
}

}  // namespace

void build_probe(laq_ctx* ctx, const int64_t* d_pk64, const int32_t* d_pk32, int64_t n, Probe& out,
                 const std::string& what, bool pooled) {
  out = Probe();
  out.n_rows = n;
  if (n == 0) return;  // DIRECT with size 0: every probe misses
  if (n > INT32_MAX) fail(LAQ_ERR_CAPACITY, "dimension has more than 2^31 rows");
  int64_t mn, mx;
  if (d_pk64) minmax_i64(ctx, d_pk64, n, &mn, &mx);
  else minmax_i32(ctx, d_pk32, n, &mn, &mx);
  if (mn < 0) fail(LAQ_ERR_DOMAIN, "negative join key " + std::to_string(mn));
  const int64_t range = mx - mn + 1;
  int* dup = reinterpret_cast<int*>(ctx->d_flags + 8);
  LAQ_CUDA(cudaMemsetAsync(dup, 0, sizeof(int), ctx->stream));
  out.row_slot = dev_mem<int32_t>(n, ctx, pooled);
  const int grid = grid_for(n, 256, ctx->sm_count * 8);
  if (range <= std::max<int64_t>(4 * n, int64_t{1} << 20) && range < (int64_t{1} << 31)) {
    out.kind = PROBE_DIRECT;
    out.base = mn;
    out.size = range;
    out.rows = dev_mem<int32_t>(range, ctx, pooled);
    LAQ_CUDA(cudaMemsetAsync(out.rows.get(), 0xFF, range * sizeof(int32_t), ctx->stream));
    if (d_pk64) direct_insert<<<grid, 256, 0, ctx->stream>>>(d_pk64, n, mn, out.rows.get(), out.row_slot.get(), dup);
    else direct_insert<<<grid, 256, 0, ctx->stream>>>(d_pk32, n, mn, out.rows.get(), out.row_slot.get(), dup);
    launched(ctx);
  } else {
    int64_t cap = 1024;
    while (cap < 2 * n) cap <<= 1;
    out.kind = PROBE_HASH;
    out.size = cap;
    out.keys = dev_mem<int64_t>(cap, ctx, pooled);
    out.rows = dev_mem<int32_t>(cap, ctx, pooled);
    LAQ_CUDA(cudaMemsetAsync(out.keys.get(), 0xFF, cap * sizeof(int64_t), ctx->stream));
    LAQ_CUDA(cudaMemsetAsync(out.rows.get(), 0xFF, cap * sizeof(int32_t), ctx->stream));
    auto* k = reinterpret_cast<unsigned long long*>(out.keys.get());
    if (d_pk64) hash_insert<<<grid, 256, 0, ctx->stream>>>(d_pk64, n, cap, k, out.rows.get(), out.row_slot.get(), dup);
    else hash_insert<<<grid, 256, 0, ctx->stream>>>(d_pk32, n, cap, k, out.rows.get(), out.row_slot.get(), dup);
    launched(ctx);
  }
  LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, dup, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  if (*reinterpret_cast<int*>(ctx->h_pinned) != 0) fail(LAQ_ERR_DUPLICATE_KEY, what);
}

namespace {

// ---------------------------------------------------------------------------
// the star compaction kernel (K2, optionally fused with K3)
// ---------------------------------------------------------------------------

template <class K>
struct StarArgs {
  int n_links;
  int64_t n;
  const K* fk[kMaxLinks];
  ProbeView probe[kMaxLinks];
  // outputs (each optional)
  int64_t* survivors;
  int64_t* rows64[kMaxLinks];
  int32_t* rows32[kMaxLinks];
  // fused predict (l <= 8): y[m*l + c] = sum_j partial[j][row_j*l + c]
  const double* partial[kMaxLinks];
  int64_t l;
  double* y;
  // decoupled look-back
  unsigned long long* tile_state;
  int* tile_counter;
  int64_t* nnz;  // device: total survivors (written by the last tile)
  int64_t n_tiles;
  int* err;      // bit 0: negative key among live rows
};

#define kFlagAgg (1ull << 62)
#define kFlagInc (2ull << 62)
#define kValMask ((1ull << 62) - 1)

template <class K>
__device__ __forceinline__ void load_keys(const K* __restrict__ p, int64_t row0, int64_t n, int64_t (&k)[kItems]) {
  if (row0 + kItems <= n && (reinterpret_cast<uintptr_t>(p + row0) & 15) == 0) {
    if constexpr (sizeof(K) == 4) {
      const int4 a = __ldcs(reinterpret_cast<const int4*>(p + row0));
      const int4 b = __ldcs(reinterpret_cast<const int4*>(p + row0) + 1);
      k[0] = a.x; k[1] = a.y; k[2] = a.z; k[3] = a.w; k[4] = b.x; k[5] = b.y; k[6] = b.z; k[7] = b.w;
    } else {
#pragma unroll
      for (int i = 0; i < kItems; i += 2) {
        const longlong2 v = __ldcs(reinterpret_cast<const longlong2*>(p + row0 + i));
        k[i] = v.x;
        k[i + 1] = v.y;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < kItems; ++i) k[i] = row0 + i < n ? static_cast<int64_t>(p[row0 + i]) : -1;
  }
}

// Decoupled look-back, split so the aggregate is published as soon as the
// tile's own count is known and the walk happens after independent work.
__device__ __forceinline__ void publish_aggregate(unsigned long long* state, int64_t tile, unsigned long long total) {
  atomicExch(state + tile, (tile == 0 ? kFlagInc : kFlagAgg) | total);
}

// Whole-warp walk: 32 predecessors inspected per step; the first one holding
// an inclusive prefix ends it.  Returns the exclusive prefix on every lane
// and publishes this tile's inclusive prefix.
__device__ __forceinline__ unsigned long long resolve_prefix(unsigned long long* state, int64_t tile,
                                                             unsigned long long total) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) return 0;
  unsigned long long prefix = 0;
  int64_t p = tile - 1;
  while (true) {
    const int64_t idx = p - lane;
    unsigned long long s;
    do {
      s = idx >= 0 ? *reinterpret_cast<volatile unsigned long long*>(state + idx) : kFlagInc;
    } while (!__all_sync(0xffffffffu, (s & ~kValMask) != 0));
    const unsigned inc = __ballot_sync(0xffffffffu, (s & ~kValMask) == kFlagInc);
    const int stop = inc ? __ffs(inc) - 1 : 31;  // lanes 0..stop contribute
    unsigned long long v = lane <= stop ? (s & kValMask) : 0;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    prefix += v;
    if (inc) break;
    p -= 32;
  }
  if (lane == 0) atomicExch(state + tile, kFlagInc | (prefix + total));
  return prefix;
}

// Persistent: CTAs pull tiles from an atomic counter (so every predecessor of
// a claimed tile is already running), probe, rank survivors locally, publish
// the tile aggregate, compute the predictions into shared memory (l == 1)
// while predecessors publish, resolve the prefix, then write the compacted
// output in coalesced runs.
template <class K, int NL, bool kPredict>
__global__ void __launch_bounds__(kBlock) star_kernel(const StarArgs<K> a) {
  using Scan = cub::BlockScan<int, kBlock>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ int64_t s_tile;
  __shared__ unsigned long long s_prefix;
  __shared__ double s_y[kPredict ? kTile : 1];
  const bool stage_y = kPredict && a.l == 1;

  int neg = 0;
  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(a.tile_counter, 1);
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= a.n_tiles) break;
    const int64_t row0 = tile * kTile + static_cast<int64_t>(threadIdx.x) * kItems;

    int32_t rows[NL][kItems];
    bool alive[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) alive[i] = row0 + i < a.n;
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      int64_t keys[kItems];
      load_keys<K>(a.fk[j], row0, a.n, keys);
      const ProbeView pv = a.probe[j];
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        int32_t r = -1;
        if (alive[i]) {
          neg |= keys[i] < 0 ? 1 : 0;
          r = pv.row(keys[i]);
          alive[i] = r >= 0;
        }
        rows[j][i] = r;
      }
    }

    int count = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) count += alive[i] ? 1 : 0;
    int excl, total;
    Scan(scan_tmp).ExclusiveSum(count, excl, total);
    if (threadIdx.x == 0) publish_aggregate(a.tile_state, tile, static_cast<unsigned long long>(total));

    if (stage_y) {  // predictions need only the local rank
      int local = excl;
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        if (!alive[i]) continue;
        double acc = __dadd_rn(0.0, __ldg(a.partial[0] + rows[0][i]));  // 0 + 1*x (spmm_dense)
#pragma unroll
        for (int j = 1; j < NL; ++j) acc = __dadd_rn(acc, __ldg(a.partial[j] + rows[j][i]));
        s_y[local++] = acc;
      }
    }
    if (threadIdx.x < 32) {
      const unsigned long long prefix = resolve_prefix(a.tile_state, tile, static_cast<unsigned long long>(total));
      if (threadIdx.x == 0) {
        s_prefix = prefix;
        if (tile == a.n_tiles - 1) *a.nnz = static_cast<int64_t>(prefix) + total;
      }
    }
    __syncthreads();
    const int64_t prefix = static_cast<int64_t>(s_prefix);
    if (stage_y)
      for (int t = threadIdx.x; t < total; t += kBlock) __stcs(a.y + prefix + t, s_y[t]);

    int64_t pos = prefix + excl;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      if (!alive[i]) continue;
      if (a.survivors) a.survivors[pos] = row0 + i;
#pragma unroll
      for (int j = 0; j < NL; ++j) {
        if (a.rows64[j]) a.rows64[j][pos] = rows[j][i];
        if (a.rows32[j]) a.rows32[j][pos] = rows[j][i];
      }
      if constexpr (kPredict) {
        if (!stage_y) {
          for (int64_t c = 0; c < a.l; ++c) {
            double acc = __dadd_rn(0.0, __ldg(a.partial[0] + static_cast<int64_t>(rows[0][i]) * a.l + c));
#pragma unroll
            for (int j = 1; j < NL; ++j)
              acc = __dadd_rn(acc, __ldg(a.partial[j] + static_cast<int64_t>(rows[j][i]) * a.l + c));
            __stcs(a.y + pos * a.l + c, acc);
          }
        }
      }
      ++pos;
    }
    __syncthreads();  // s_tile / s_y / scan storage are reused by the next tile
  }
  if (neg) atomicOr(a.err, 1);
}

// ---------------------------------------------------------------------------
// apply_fused_linear over explicit row maps (fusion.cpp:64-77)
// ---------------------------------------------------------------------------

template <class I>
struct ApplyArgs {
  int n_parts;
  int64_t rows;
  int64_t l;
  const I* idx[kMaxLinks];
  const double* partial[kMaxLinks];
  double* out;
};

// l <= 8: one thread per target row.
template <class I>
__global__ void apply_rows_kernel(const ApplyArgs<I> a) {
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < a.rows; m += (int64_t)gridDim.x * blockDim.x) {
    int64_t r[kMaxLinks];
    for (int j = 0; j < a.n_parts; ++j) r[j] = static_cast<int64_t>(a.idx[j][m]);
    for (int64_t c = 0; c < a.l; ++c) {
      double acc = __dadd_rn(0.0, __ldg(a.partial[0] + r[0] * a.l + c));  // 0 + 1*x (spmm_dense)
      for (int j = 1; j < a.n_parts; ++j) acc = __dadd_rn(acc, __ldg(a.partial[j] + r[j] * a.l + c));
      __stcs(a.out + m * a.l + c, acc);
    }
  }
}

// l > 8: one warp per target row, lanes across the output width.
template <class I>
__global__ void apply_warp_kernel(const ApplyArgs<I> a) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t m = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; m < a.rows; m += warps) {
    int64_t r[kMaxLinks];
    for (int j = 0; j < a.n_parts; ++j) r[j] = static_cast<int64_t>(a.idx[j][m]);
    for (int64_t c = lane; c < a.l; c += 32) {
      double acc = __dadd_rn(0.0, __ldg(a.partial[0] + r[0] * a.l + c));  // 0 + 1*x (spmm_dense)
      for (int j = 1; j < a.n_parts; ++j) acc = __dadd_rn(acc, __ldg(a.partial[j] + r[j] * a.l + c));
      __stcs(a.out + m * a.l + c, acc);
    }
  }
}

template <class I>
void launch_apply(laq_ctx* ctx, const ApplyArgs<I>& a) {
  if (a.rows == 0 || a.l == 0) return;
  if (a.l <= 8) {
    apply_rows_kernel<I><<<grid_for(a.rows, 256, ctx->sm_count * 16), 256, 0, ctx->stream>>>(a);
  } else {
    apply_warp_kernel<I><<<grid_for(a.rows, 8, ctx->sm_count * 16), 256, 0, ctx->stream>>>(a);
  }
  launched(ctx);
}

// ---------------------------------------------------------------------------
// materialize (laqops.cpp:338-374): T[m, tgt] = B_j[i_j[m], src]
// ---------------------------------------------------------------------------

__global__ void materialize_kernel(const int64_t* __restrict__ idx, int64_t rows, const double* __restrict__ dim,
                                   int64_t dim_cols, const int32_t* __restrict__ place, int64_t k,
                                   double* __restrict__ out) {
  const int64_t total = rows * dim_cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = e / dim_cols, c = e - m * dim_cols;
    out[m * k + place[c]] = __dadd_rn(0.0, __ldg(dim + idx[m] * dim_cols + c));  // target += 1*x
  }
}

}  // namespace

// Lookback scratch sized for n fact rows.
struct StarScratch {
  DevMem<unsigned long long> tile_state;
  DevMem<int> counter;
  int64_t cap_tiles = 0;
  void ensure(int64_t tiles) {
    if (tiles <= cap_tiles) return;
    tile_state = DevMem<unsigned long long>(tiles);
    counter = DevMem<int>(1);
    cap_tiles = tiles;
  }
};

template <class K>
void run_star(laq_ctx* ctx, StarArgs<K>& a, StarScratch& scratch, bool predict) {
  a.n_tiles = (a.n + kTile - 1) / kTile;
  if (a.n_tiles == 0) {
    LAQ_CUDA(cudaMemsetAsync(a.nnz, 0, sizeof(int64_t), ctx->stream));
    return;
  }
  scratch.ensure(a.n_tiles);
  a.tile_state = scratch.tile_state.get();
  a.tile_counter = scratch.counter.get();
  LAQ_CUDA(cudaMemsetAsync(a.tile_state, 0, a.n_tiles * sizeof(unsigned long long), ctx->stream));
  LAQ_CUDA(cudaMemsetAsync(a.tile_counter, 0, sizeof(int), ctx->stream));
  // Persistent grid: a few resident CTAs per SM pull tiles dynamically.
  const unsigned g = static_cast<unsigned>(std::min<int64_t>(a.n_tiles, int64_t{ctx->sm_count} * 6));
  cudaStream_t s = ctx->stream;
#define LAQ_STAR_CASE(N)                                                   \
  case N:                                                                  \
    if (predict) star_kernel<K, N, true><<<g, kBlock, 0, s>>>(a);          \
    else star_kernel<K, N, false><<<g, kBlock, 0, s>>>(a);                 \
    break;
  switch (a.n_links) {
    LAQ_STAR_CASE(1) LAQ_STAR_CASE(2) LAQ_STAR_CASE(3) LAQ_STAR_CASE(4)
    LAQ_STAR_CASE(5) LAQ_STAR_CASE(6) LAQ_STAR_CASE(7) LAQ_STAR_CASE(8)
    default: fail(LAQ_ERR_UNSUPPORTED, "star join supports 1..8 dimensions");
  }
#undef LAQ_STAR_CASE
  launched(ctx);
}

// Host-buffer pipeline of laq_probe_fused_predict_host: fact keys H2D on
// `up`, the fused predict on the context stream, predictions D2H on `down`,
// double-buffered so chunk c+1's keys and chunk c-1's predictions cross PCIe
// (full duplex) while chunk c is probed.
struct HostPipe {
  cudaStream_t up = nullptr, down = nullptr;
  cudaEvent_t loaded[2]{}, computed[2]{}, drained[2]{};
  DevMem<int32_t> keys[2];  // [link][cap] per buffer
  DevMem<double> y[2];      // [cap][l] per buffer
  DevMem<int64_t> nnz;      // survivors per chunk
  int64_t* h_nnz = nullptr;  // pinned copy of nnz
  int64_t cap = 0, chunks = 0;
  int nl = 0, l = 0;
  HostPipe() {
    LAQ_CUDA(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking));
    LAQ_CUDA(cudaStreamCreateWithFlags(&down, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b)
      for (cudaEvent_t* e : {&loaded[b], &computed[b], &drained[b]})
        LAQ_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  ~HostPipe() {
    for (int b = 0; b < 2; ++b)
      for (cudaEvent_t e : {loaded[b], computed[b], drained[b]}) cudaEventDestroy(e);
    if (up) cudaStreamDestroy(up);
    if (down) cudaStreamDestroy(down);
    if (h_nnz) cudaFreeHost(h_nnz);
  }
};

}  // namespace laq

using namespace laq;

struct laq_probe {
  int n_links = 0;
  Probe probes[kMaxLinks];
  StarScratch scratch;
  DevMem<int> err;
  // slot-ordered partials + existence bitmaps (predict_slot.cuh), rebuilt per call
  DevMem<double> pslot[kMaxLinks];
  DevMem<uint32_t> bits[kMaxLinks];
  int64_t pslot_l = 0;
  bool bound = false;
  // chunk counts / offsets (scan_chunks_kernel)
  DevMem<int> chunk_counts;
  DevMem<int64_t> chunk_offsets;
  int64_t chunk_cap = 0;
  // optimistic single pass: [0] chunks with a missing key (counted by the
  // direct pass, moved to [1] and cleared by the scan pass), [1] the decision
  // the write pass reads
  // [2] CTAs finished (the one-launch form's last-CTA counter, reset by that CTA)
  DevMem<unsigned long long> miss{3};
  std::unique_ptr<HostPipe> host;  // laq_probe_fused_predict_host's streams and buffers
  bool tables_stable = false;      // staged tables unchanged since the last one-launch predict (PDL is safe)
};

namespace laq {
int probe_links(const laq_probe* p) { return p->n_links; }
ProbeView probe_view(const laq_probe* p, int j) { return p->probes[j].view(); }
}  // namespace laq


namespace laq {
namespace {

// Slot-ordered partials + existence bitmaps for every link (predict_slot.cuh).
void bind_slots(laq_ctx* ctx, laq_probe* p, const double* const* d_P, int64_t l) {
  for (int j = 0; j < p->n_links; ++j) {
    const Probe& pr = p->probes[j];
    const int64_t size = pr.size;
    // padded to 16-byte granules (TMA bulk staging, run_slot_predict)
    const int64_t words = (std::max<int64_t>(1, (size + 31) / 32) + 3) & ~int64_t{3};
    const int64_t doubles = (std::max<int64_t>(size * l, 1) + 1) & ~int64_t{1};
    if (p->pslot_l != l || p->pslot[j].n < static_cast<size_t>(doubles) || p->bits[j].n < static_cast<size_t>(words)) {
      p->pslot[j] = DevMem<double>(static_cast<size_t>(doubles));
      p->bits[j] = DevMem<uint32_t>(static_cast<size_t>(words));
    }
    LAQ_CUDA(cudaMemsetAsync(p->bits[j].get(), 0, words * sizeof(uint32_t), ctx->stream));
    if (pr.n_rows > 0) {
      slot::scatter_slots_kernel<<<grid_for(pr.n_rows, 256, ctx->sm_count * 4), 256, 0, ctx->stream>>>(
          pr.row_slot.get(), pr.n_rows, d_P[j], l, p->pslot[j].get(), p->bits[j].get());
      launched(ctx);
    }
  }
  p->pslot_l = l;
  p->bound = true;
  p->tables_stable = false;  // the bind kernels just wrote the staged tables: the next predict launches normally
}

// Fused predict over slot-ordered partials; every probe must be DIRECT.
// d_P == nullptr uses the partials bound by laq_probe_bind_partials.
void run_slot_predict(laq_ctx* ctx, laq_probe* p, const int32_t* const* d_fks, int64_t n, const double* const* d_P,
                      int64_t l, double* d_out, int64_t* d_survivors, int64_t* d_nnz) {
  slot::Args a{};
  a.n = n;
  a.l = l;
  int64_t words_total = 0;
  if (d_P) bind_slots(ctx, p, d_P, l);
  else if (!p->bound || p->pslot_l != l) fail(LAQ_ERR_SHAPE, "fused predict: no partials bound for this output width");
  for (int j = 0; j < p->n_links; ++j) {
    const Probe& pr = p->probes[j];
    a.fk[j] = d_fks[j];
    a.base[j] = pr.base;
    a.size[j] = pr.size;
    a.bits[j] = p->bits[j].get();
    a.pslot[j] = p->pslot[j].get();
    a.bits_off[j] = -1;
    a.p_off[j] = -1;
  }
  // Shared-memory staging of the existence bitmaps that fit (partials are
  // gathered through L1: high occupancy matters more than staging them).
  // Tables start on 16-byte boundaries and span whole 16-byte granules (the
  // direct kernel stages them with TMA bulk copies; the sources are padded).
  int64_t bulk = 0;
  for (int j = 0; j < p->n_links; ++j) {
    const int64_t words = (std::max<int64_t>(1, (a.size[j] + 31) / 32) + 3) & ~int64_t{3};
    if ((words_total + words) * 4 <= 32 * 1024) {
      a.bits_off[j] = static_cast<int>(words_total);
      a.bits_bytes[j] = static_cast<int>(words * 4);
      bulk += words * 4;
      words_total += words;
    }
  }
  a.smem_words = static_cast<int>(words_total);
  // l == 1: stage the slot-ordered partials too when they fit in 96 KB
  // (shared-memory gathers instead of one L1 wavefront per lane).
  int64_t doubles = 0;
  if (l == 1 && !std::getenv("LAQ_PREDICT_NO_PSTAGE"))
    for (int j = 0; j < p->n_links; ++j) {
      const int64_t d = (std::max<int64_t>(a.size[j], 1) + 1) & ~int64_t{1};
      if ((doubles + d) * 8 <= 96 * 1024) {
        a.p_off[j] = static_cast<int>(doubles);
        a.p_bytes[j] = static_cast<int>(d * 8);
        bulk += d * 8;
        doubles += d;
      }
    }
  a.smem_doubles = static_cast<int>(doubles);
  a.bulk_bytes = std::getenv("LAQ_PREDICT_NO_BULK") ? 0 : static_cast<int>(bulk);
  a.y = d_out;
  a.survivors = d_survivors;
  a.nnz = d_nnz;
  const int64_t n_chunks = (n + slot::kChunkRows - 1) / slot::kChunkRows;
  if (n_chunks == 0) {
    LAQ_CUDA(cudaMemsetAsync(d_nnz, 0, sizeof(int64_t), ctx->stream));
    return;
  }
  if (p->chunk_cap < n_chunks) {
    p->chunk_counts = DevMem<int>(n_chunks);
    p->chunk_offsets = DevMem<int64_t>(n_chunks);
    p->chunk_cap = n_chunks;
  }
  const size_t smem = static_cast<size_t>(words_total) * 4;
  const size_t smem_w = static_cast<size_t>((words_total * 4 + 15) & ~int64_t{15}) + static_cast<size_t>(doubles) * 8;
  // l == 1 and no LAQ_PREDICT_TWO_PASS: optimistic single pass + device-decided
  // compaction fallback (direct_chunks_kernel); otherwise count + scan + write.
  const bool optimistic = l == 1 && !std::getenv("LAQ_PREDICT_TWO_PASS");
  // Small inputs (<= 4M rows): one launch per call (launch latency dominates
  // there: 1M rows = 12 MB = 1.8 us of HBM time); the miss path is compacted by
  // the last CTA.  LAQ_PREDICT_ONE_LAUNCH=0 keeps the three-launch form.
  const char* ol = std::getenv("LAQ_PREDICT_ONE_LAUNCH");
  const bool one_launch = optimistic && n_chunks <= 4096 && !(ol && std::string(ol) == "0");
  constexpr int64_t kOneChunkRows = 256;
  unsigned long long* miss = p->miss.get();
  unsigned long long* decision = p->miss.get() + 1;
  auto launch = [&](auto count_k, auto direct_k, auto direct_small_k, auto direct_one_k, auto write_k) {
    LAQ_CUDA(cudaFuncSetAttribute(write_k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_w)));
    const int64_t want = (n_chunks + slot::kWarpThreads / 32 - 1) / (slot::kWarpThreads / 32);
    int per_sm = 0;
    // Large inputs: one 1024-thread CTA per SM (one staged copy of the partials,
    // 32 warps/SM; 1e8 rows 0.278 -> 0.218 ms).  Below two chunks per warp of
    // such a grid, 256-thread CTAs spread the chunks over every SM instead.
    const bool big = n_chunks >= int64_t{ctx->sm_count} * (slot::kDirectBT / 32) * 2;
    if (optimistic && big) {
      LAQ_CUDA(cudaFuncSetAttribute(direct_k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_w)));
      const unsigned g0 = static_cast<unsigned>(ctx->sm_count);
      direct_k<<<g0, slot::kDirectBT, smem_w, ctx->stream>>>(a, n_chunks, p->chunk_counts.get(), miss, nullptr,
                                                              nullptr);
    } else if (optimistic) {
      LAQ_CUDA(cudaFuncSetAttribute(direct_small_k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_w)));
      LAQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, direct_small_k, slot::kWarpThreads, smem_w));
      const unsigned g0 = static_cast<unsigned>(std::min<int64_t>(want, int64_t{ctx->sm_count} * std::max(per_sm, 1)));
      if (one_launch) {  // the whole call in one launch: the last CTA decides (and compacts on a miss)
        // 1024-thread CTAs (one staged copy of the tables per SM) over 256-row
        // chunks (1M rows = 3.9K chunks: every warp of the grid gets one).
        const int64_t chunks1 = (n + kOneChunkRows - 1) / kOneChunkRows;
        if (p->chunk_cap < chunks1) {
          p->chunk_counts = DevMem<int>(chunks1);
          p->chunk_offsets = DevMem<int64_t>(chunks1);
          p->chunk_cap = chunks1;
        }
        LAQ_CUDA(cudaFuncSetAttribute(direct_one_k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_w)));
        const unsigned g1 = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((chunks1 + 31) / 32, ctx->sm_count)));
        // Programmatic dependent launch once the staged tables are stable (no
        // bind since the previous call): this call's table staging overlaps the
        // previous kernel's tail; it waits (griddepcontrol.wait) before reading
        // keys or writing anything.  LAQ_PREDICT_PDL=0 disables.
        const char* pdl_env = std::getenv("LAQ_PREDICT_PDL");
        const bool pdl = p->tables_stable && !(pdl_env && std::string(pdl_env) == "0");
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(g1);
        cfg.blockDim = dim3(slot::kDirectBT);
        cfg.dynamicSmemBytes = smem_w;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 1 : 0;
        LAQ_CUDA(cudaLaunchKernelEx(&cfg, direct_one_k, a, static_cast<int64_t>(chunks1), p->chunk_counts.get(), miss,
                                    p->miss.get() + 2, p->chunk_offsets.get()));
        p->tables_stable = true;
        return;
      }
      direct_small_k<<<g0, slot::kWarpThreads, smem_w, ctx->stream>>>(a, n_chunks, p->chunk_counts.get(), miss,
                                                                      nullptr, nullptr);
    } else {
      LAQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, count_k, slot::kWarpThreads, smem));
      const unsigned g1 = static_cast<unsigned>(std::min<int64_t>(want, int64_t{ctx->sm_count} * std::max(per_sm, 1)));
      count_k<<<g1, slot::kWarpThreads, smem, ctx->stream>>>(a, n_chunks, p->chunk_counts.get());
    }
    LAQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, write_k, slot::kWarpThreads, smem_w));
    const unsigned g2 = static_cast<unsigned>(std::min<int64_t>(want, int64_t{ctx->sm_count} * std::max(per_sm, 1)));
    slot::scan_chunks_kernel<<<1, slot::kScanThreads, 0, ctx->stream>>>(
        p->chunk_counts.get(), n_chunks, p->chunk_offsets.get(), optimistic ? miss : nullptr, decision);
    write_k<<<g2, slot::kWarpThreads, smem_w, ctx->stream>>>(a, n_chunks, p->chunk_offsets.get(),
                                                             optimistic ? decision : nullptr);
    ctx->launches += 2;
  };
  switch (p->n_links) {
#define LAQ_SLOT_CASE(N) \
    case N: launch(slot::count_chunks_kernel<N>, slot::direct_chunks_kernel<N, slot::kDirectBT>, \
                   slot::direct_chunks_kernel<N, slot::kWarpThreads>, \
                   slot::direct_chunks_kernel<N, slot::kDirectBT, kOneChunkRows / slot::kSegRows>, \
                   slot::write_chunks_kernel<N>); break;
    LAQ_SLOT_CASE(1) LAQ_SLOT_CASE(2) LAQ_SLOT_CASE(3) LAQ_SLOT_CASE(4)
    LAQ_SLOT_CASE(5) LAQ_SLOT_CASE(6) LAQ_SLOT_CASE(7) LAQ_SLOT_CASE(8)
#undef LAQ_SLOT_CASE
    default: fail(LAQ_ERR_UNSUPPORTED, "fused predict supports 1..8 dimensions");
  }
  launched(ctx);
}

}  // namespace
}  // namespace laq

extern "C" {

int laq_star_join(laq_ctx* ctx, int32_t n_links, const int64_t* const* d_fks, int64_t n_fact,
                  const int64_t* const* d_pks, const int64_t* h_pk_rows, int64_t* d_survivors,
                  int64_t* const* d_dim_rows, int64_t* h_nnz) {
  return guard(ctx, [&] {
    if (n_links < 0 || n_links > kMaxLinks) fail(LAQ_ERR_UNSUPPORTED, "star join supports up to 8 dimensions");
    if (n_links == 0) {  // nothing to join: every fact row survives
      *h_nnz = n_fact;
      fail(LAQ_ERR_UNSUPPORTED, "star join with no dimensions");
    }
    Probe probes[kMaxLinks];
    for (int j = 0; j < n_links; ++j)
      build_probe(ctx, d_pks[j], nullptr, h_pk_rows[j], probes[j], "multiway_star_join: duplicate keys in dim " + std::to_string(j),
                  /*pooled=*/true);
    StarArgs<int64_t> a{};
    a.n_links = n_links;
    a.n = n_fact;
    for (int j = 0; j < n_links; ++j) {
      a.fk[j] = d_fks[j];
      a.probe[j] = probes[j].view();
      a.rows64[j] = d_dim_rows ? d_dim_rows[j] : nullptr;
    }
    a.survivors = d_survivors;
    a.nnz = ctx->d_flags + 16;
    a.err = reinterpret_cast<int*>(ctx->d_flags + 17);
    LAQ_CUDA(cudaMemsetAsync(a.err, 0, sizeof(int), ctx->stream));
    StarScratch scratch;
    run_star(ctx, a, scratch, false);
    LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, ctx->d_flags + 16, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    if (ctx->h_pinned[1] & 1) fail(LAQ_ERR_DOMAIN, "negative join key");
    *h_nnz = ctx->h_pinned[0];
  });
}

int laq_probe_build(laq_ctx* ctx, int32_t n_links, const int32_t* const* d_pks, const int64_t* h_pk_rows,
                    laq_probe** out) {
  return guard(ctx, [&] {
    if (n_links < 1 || n_links > kMaxLinks) fail(LAQ_ERR_UNSUPPORTED, "fused star predict supports 1..8 dimensions");
    auto* p = new laq_probe();
    LAQ_CUDA(cudaMemset(p->miss.get(), 0, 3 * sizeof(unsigned long long)));
    try {
      p->n_links = n_links;
      for (int j = 0; j < n_links; ++j)
        build_probe(ctx, nullptr, d_pks[j], h_pk_rows[j], p->probes[j],
                    "multiway_star_join: duplicate keys in dim " + std::to_string(j));
      p->err = DevMem<int>(1);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

int laq_probe_join_rows(laq_ctx* ctx, const laq_probe* probe, const int32_t* const* d_fks, int64_t n_fact,
                        int32_t* const* d_rows, int64_t* d_survivors, int64_t* d_nnz) {
  return guard(ctx, [&] {
    auto* p = const_cast<laq_probe*>(probe);
    StarArgs<int32_t> a{};
    a.n_links = p->n_links;
    a.n = n_fact;
    for (int j = 0; j < p->n_links; ++j) {
      a.fk[j] = d_fks[j];
      a.probe[j] = p->probes[j].view();
      a.rows32[j] = d_rows[j];
    }
    a.survivors = d_survivors;
    a.nnz = d_nnz;
    a.err = p->err.get();
    run_star(ctx, a, p->scratch, false);
  });
}

int laq_probe_destroy(laq_probe* p) {
  delete p;
  return LAQ_OK;
}

int laq_probe_bind_partials(laq_ctx* ctx, laq_probe* p, const double* const* d_partials, int64_t l) {
  return guard(ctx, [&] {
    if (l < 1) fail(LAQ_ERR_SHAPE, "bind_partials: output width must be positive");
    for (int j = 0; j < p->n_links; ++j)
      if (p->probes[j].kind != PROBE_DIRECT) fail(LAQ_ERR_UNSUPPORTED, "bind_partials: hashed dimension keys");
    bind_slots(ctx, p, d_partials, l);
  });
}

int laq_probe_fused_predict(laq_ctx* ctx, const laq_probe* probe, const int32_t* const* d_fks, int64_t n_fact,
                            const double* const* d_partials, int64_t l, double* d_out, int64_t* d_survivors,
                            int64_t* d_nnz) {
  return guard(ctx, [&] {
    if (l < 1 || l > 8) fail(LAQ_ERR_UNSUPPORTED, "fused single-pass predict handles l <= 8 (use star join + apply)");
    auto* p = const_cast<laq_probe*>(probe);
    bool all_direct = !std::getenv("LAQ_PREDICT_GENERIC");
    for (int j = 0; j < p->n_links; ++j) all_direct = all_direct && p->probes[j].kind == PROBE_DIRECT;
    if (all_direct) {
      run_slot_predict(ctx, p, d_fks, n_fact, d_partials, l, d_out, d_survivors, d_nnz);
      return;
    }
    if (!d_partials) fail(LAQ_ERR_SHAPE, "fused predict: partials required for hashed dimension keys");
    StarArgs<int32_t> a{};
    a.n_links = p->n_links;
    a.n = n_fact;
    for (int j = 0; j < p->n_links; ++j) {
      a.fk[j] = d_fks[j];
      a.probe[j] = p->probes[j].view();
      a.partial[j] = d_partials[j];
    }
    a.l = l;
    a.y = d_out;
    a.survivors = d_survivors;
    a.nnz = d_nnz;
    a.err = p->err.get();
    run_star(ctx, a, p->scratch, true);
  });
}

int laq_probe_fused_predict_host(laq_ctx* ctx, const laq_probe* probe, const int32_t* const* h_fks, int64_t n_fact,
                                 int64_t l, double* h_out, int64_t chunk_rows, int64_t* h_nnz) {
  return guard(ctx, [&] {
    auto* p = const_cast<laq_probe*>(probe);
    if (l < 1 || l > 8) fail(LAQ_ERR_UNSUPPORTED, "fused single-pass predict handles l <= 8 (use star join + apply)");
    for (int j = 0; j < p->n_links; ++j)
      if (p->probes[j].kind != PROBE_DIRECT)
        fail(LAQ_ERR_UNSUPPORTED, "host-buffer fused predict: hashed dimension keys (use laq_probe_fused_predict)");
    if (!p->bound || p->pslot_l != l) fail(LAQ_ERR_SHAPE, "host-buffer fused predict: bind the partials first");
    if (n_fact < 0) fail(LAQ_ERR_SHAPE, "negative row count");
    // Default: one piece up to 4M rows (PCIe runs H2D and D2H only partly in
    // parallel on these boxes: 4 MB up + 8 MB down take 197 us concurrently vs
    // 231 us back to back, less than the per-piece stream/event overhead at that
    // size), eight pieces above.
    if (chunk_rows <= 0) chunk_rows = n_fact <= (int64_t{4} << 20) ? n_fact : (n_fact + 7) / 8;
    chunk_rows = std::max<int64_t>(1024, (chunk_rows + 1023) & ~int64_t{1023});  // 16-byte aligned key pieces
    const int64_t chunks = std::max<int64_t>(1, (n_fact + chunk_rows - 1) / chunk_rows);
    if (!p->host) p->host = std::make_unique<HostPipe>();
    HostPipe& h = *p->host;
    if (h.cap < chunk_rows || h.nl != p->n_links || h.l != l) {
      for (int b = 0; b < 2; ++b) {
        h.keys[b] = DevMem<int32_t>(static_cast<size_t>(chunk_rows * p->n_links));
        h.y[b] = DevMem<double>(static_cast<size_t>(chunk_rows * l));
      }
      h.cap = chunk_rows, h.nl = p->n_links, h.l = static_cast<int>(l);
    }
    if (h.chunks < chunks) {
      h.nnz = DevMem<int64_t>(static_cast<size_t>(chunks));
      if (h.h_nnz) cudaFreeHost(h.h_nnz);
      h.h_nnz = nullptr;
      LAQ_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h.h_nnz), chunks * sizeof(int64_t)));
      h.chunks = chunks;
    }
    if (chunks == 1) {  // one piece: H2D, probe, D2H in order on the context stream
      const int32_t* kp[kMaxLinks];
      for (int j = 0; j < p->n_links; ++j) {
        int32_t* d = h.keys[0].get() + j * h.cap;
        if (n_fact > 0)
          LAQ_CUDA(cudaMemcpyAsync(d, h_fks[j], n_fact * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
        kp[j] = d;
      }
      run_slot_predict(ctx, p, kp, n_fact, nullptr, l, h.y[0].get(), nullptr, h.nnz.get());
      if (n_fact > 0)
        LAQ_CUDA(cudaMemcpyAsync(h_out, h.y[0].get(), n_fact * l * sizeof(double), cudaMemcpyDeviceToHost,
                                 ctx->stream));
      LAQ_CUDA(cudaMemcpyAsync(h.h_nnz, h.nnz.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
      sync(ctx);
      *h_nnz = h.h_nnz[0];
      return;
    }
    // the copies may not start before earlier work on the context stream
    LAQ_CUDA(cudaEventRecord(h.computed[1], ctx->stream));
    LAQ_CUDA(cudaStreamWaitEvent(h.up, h.computed[1], 0));
    for (int64_t c = 0; c < chunks; ++c) {
      const int b = static_cast<int>(c & 1);
      const int64_t r0 = c * chunk_rows, m = std::min(chunk_rows, n_fact - r0);
      if (c >= 2) LAQ_CUDA(cudaStreamWaitEvent(h.up, h.drained[b], 0));  // buffer b's previous chunk is out
      const int32_t* kp[kMaxLinks];
      for (int j = 0; j < p->n_links; ++j) {
        int32_t* d = h.keys[b].get() + j * h.cap;
        if (m > 0) LAQ_CUDA(cudaMemcpyAsync(d, h_fks[j] + r0, m * sizeof(int32_t), cudaMemcpyHostToDevice, h.up));
        kp[j] = d;
      }
      LAQ_CUDA(cudaEventRecord(h.loaded[b], h.up));
      LAQ_CUDA(cudaStreamWaitEvent(ctx->stream, h.loaded[b], 0));
      run_slot_predict(ctx, p, kp, m, nullptr, l, h.y[b].get(), nullptr, h.nnz.get() + c);
      LAQ_CUDA(cudaEventRecord(h.computed[b], ctx->stream));
      LAQ_CUDA(cudaStreamWaitEvent(h.down, h.computed[b], 0));
      if (m > 0)
        LAQ_CUDA(cudaMemcpyAsync(h_out + r0 * l, h.y[b].get(), m * l * sizeof(double), cudaMemcpyDeviceToHost,
                                 h.down));
      LAQ_CUDA(cudaEventRecord(h.drained[b], h.down));
    }
    LAQ_CUDA(cudaMemcpyAsync(h.h_nnz, h.nnz.get(), chunks * sizeof(int64_t), cudaMemcpyDeviceToHost, h.down));
    LAQ_CUDA(cudaStreamSynchronize(h.down));
    // Each chunk's survivors sit at its own start: close the gaps (none when
    // every key joins, the common case) keeping ascending fact order.
    int64_t at = 0;
    for (int64_t c = 0; c < chunks; ++c) {
      const int64_t r0 = c * chunk_rows, k = h.h_nnz[c];
      if (at != r0 && k > 0) std::memmove(h_out + at * l, h_out + r0 * l, static_cast<size_t>(k * l) * sizeof(double));
      at += k;
    }
    *h_nnz = at;
  });
}

int laq_fused_star_predict(laq_ctx* ctx, int32_t n_links, const int32_t* const* d_fks, int64_t n_fact,
                           const int32_t* const* d_pks, const int64_t* h_pk_rows, const double* const* d_partials,
                           int64_t l, double* d_out, int64_t* d_survivors, int64_t* h_nnz) {
  laq_probe* p = nullptr;
  int rc = laq_probe_build(ctx, n_links, d_pks, h_pk_rows, &p);
  if (rc) return rc;
  rc = guard(ctx, [&] {
    if (l <= 8) {
      int rc2 = laq_probe_fused_predict(ctx, p, d_fks, n_fact, d_partials, l, d_out, d_survivors, ctx->d_flags + 20);
      if (rc2) fail(rc2, ctx->err);
    } else {
      // Wide outputs: compaction pass writing int32 row maps, then the warp-wide gather-sum.
      StarArgs<int32_t> a{};
      a.n_links = n_links;
      a.n = n_fact;
      std::vector<DevBuf<int32_t>> maps;
      for (int j = 0; j < n_links; ++j) {
        maps.emplace_back(ctx, static_cast<size_t>(std::max<int64_t>(n_fact, 1)));
        a.fk[j] = d_fks[j];
        a.probe[j] = p->probes[j].view();
        a.rows32[j] = maps.back().get();
      }
      a.survivors = d_survivors;
      a.nnz = ctx->d_flags + 20;
      a.err = p->err.get();
      run_star(ctx, a, p->scratch, false);
      LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, ctx->d_flags + 20, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
      sync(ctx);
      ApplyArgs<int32_t> ap{};
      ap.n_parts = n_links;
      ap.rows = ctx->h_pinned[0];
      ap.l = l;
      for (int j = 0; j < n_links; ++j) {
        ap.idx[j] = maps[j].get();
        ap.partial[j] = d_partials[j];
      }
      ap.out = d_out;
      launch_apply(ctx, ap);
    }
    LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, ctx->d_flags + 20, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    *h_nnz = ctx->h_pinned[0];
  });
  laq_probe_destroy(p);
  return rc;
}

int laq_apply_fused_linear(laq_ctx* ctx, int32_t n_parts, const int64_t* const* d_idx, int64_t rows,
                           const double* const* d_partials, const int64_t* h_partial_rows, int64_t l,
                           double* d_out) {
  return guard(ctx, [&] {
    (void)h_partial_rows;
    if (n_parts < 1) fail(LAQ_ERR_SHAPE, "apply_fused_linear: map/partial list lengths");
    if (n_parts > kMaxLinks) fail(LAQ_ERR_UNSUPPORTED, "apply_fused_linear supports up to 8 partials");
    ApplyArgs<int64_t> a{};
    a.n_parts = n_parts;
    a.rows = rows;
    a.l = l;
    for (int j = 0; j < n_parts; ++j) {
      a.idx[j] = d_idx[j];
      a.partial[j] = d_partials[j];
    }
    a.out = d_out;
    launch_apply(ctx, a);
  });
}

int laq_materialize(laq_ctx* ctx, int32_t n_parts, const int64_t* const* d_idx, int64_t rows,
                    const double* const* d_dims, const int64_t* h_dim_rows, const int64_t* h_dim_cols,
                    const int64_t* const* h_placements, int64_t k, double* d_out) {
  return guard(ctx, [&] {
    (void)h_dim_rows;
    if (n_parts < 1) fail(LAQ_ERR_SHAPE, "materialize: input list lengths");
    std::vector<char> claimed(static_cast<size_t>(k), 0);
    for (int j = 0; j < n_parts; ++j)
      for (int64_t c = 0; c < h_dim_cols[j]; ++c) {
        const int64_t t = h_placements[j][c];
        if (t < 0 || t >= k) fail(LAQ_ERR_MAPPING, "column map: target index " + std::to_string(t) + " out of range");
        if (claimed[t]) fail(LAQ_ERR_MAPPING, "materialize: overlapping target column " + std::to_string(t));
        claimed[t] = 1;
      }
    if (rows == 0 || k == 0) return;
    LAQ_CUDA(cudaMemsetAsync(d_out, 0, rows * k * sizeof(double), ctx->stream));
    for (int j = 0; j < n_parts; ++j) {
      if (h_dim_cols[j] == 0) continue;
      std::vector<int32_t> pl(h_placements[j], h_placements[j] + h_dim_cols[j]);
      DevBuf<int32_t> dpl(ctx, pl.size());
      LAQ_CUDA(cudaMemcpyAsync(dpl.get(), pl.data(), pl.size() * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
      materialize_kernel<<<grid_for(rows * h_dim_cols[j], 256, ctx->sm_count * 16), 256, 0, ctx->stream>>>(
          d_idx[j], rows, d_dims[j], h_dim_cols[j], dpl.get(), k, d_out);
      launched(ctx);
      sync(ctx);  // pl (host) must outlive the async copy
    }
  });
}

}  // extern "C"
