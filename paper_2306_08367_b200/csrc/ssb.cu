// K4 ssb_scan_groupby: the query plan driver run_query_laq (cli.cpp:73-138)
// as ONE fused pass over the fact table per query.
//
// Reference plan:  filter_table(fact), filter_table(dim_j)  ->  multiway_star_join
// (one-hot key matrices x spmm per link)  ->  gather measure (spmm_dense)  ->
// groupby_sum_multi (sort-unique + segmented sum)  ->  sort_rows.
//
// Here:
//  * each dimension link owns a probe table (probe.cuh) built once per star;
//  * per query, a tiny kernel per link evaluates that link's dimension filters
//    and group attributes and writes, for every probe slot, a "code":
//    -1 = the dim row fails its filters (or the key is absent), else the
//    link's contribution to the dense group id (mixed radix over the group
//    columns' value ranges, first group column most significant, so ascending
//    group id == ascending group tuple == the order groupby_sum_multi +
//    sort_rows produce);
//  * the scan kernel streams the touched int32 fact columns once (16-20 B/row),
//    evaluates fact filters, probes each link (1 gather into an L2-resident
//    code table, skipped for rows already dead), and accumulates per group id
//    an exact int64 (count, sum) in shared memory; blocks merge with global
//    atomics into the caller's accumulator (the NCCL all-reduce buffer when
//    sharded across GPUs).
// Integer sums are exact, so results equal the reference bit for bit.
#include <algorithm>
#include <climits>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "probe.cuh"

namespace laq {
namespace {

constexpr int kMaxLinks = 8;
constexpr int kMaxFactFilters = 4;
constexpr int kMaxFactGroups = 4;
constexpr int kMaxDimFilters = 8;
constexpr int kMaxDimGroups = 4;
constexpr int kScanBlock = 256;
constexpr int64_t kSmemBins = 6144;  // group ids accumulated in shared memory

struct DevCol {
  std::string name;
  int kind = LAQ_COL_INT;
  int32_t* d = nullptr;  // int32 device column (nullptr for float columns)
  int64_t mn = 0, mx = -1;
};

struct DevTable {
  std::string name;
  int64_t rows = 0;
  std::vector<DevCol> cols;
  std::vector<DevMem<int32_t>> owned;

  const DevCol* find(const std::string& n) const {
    for (const auto& c : cols)
      if (c.name == n) return &c;
    return nullptr;
  }
};

// ---- upload: int64 -> int32 narrowing with range check and min/max ----------

__global__ void narrow_kernel(const int64_t* __restrict__ src, int32_t* __restrict__ dst, int64_t n,
                              unsigned long long* mnmx, int* overflow) {
  int64_t mn = LLONG_MAX, mx = LLONG_MIN;
  int of = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = src[i];
    of |= (v < INT32_MIN || v > INT32_MAX) ? 1 : 0;
    dst[i] = static_cast<int32_t>(v);
    mn = v < mn ? v : mn;
    mx = v > mx ? v : mx;
  }
  for (int o = 16; o; o >>= 1) {
    const int64_t a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
    of |= __shfl_xor_sync(0xffffffffu, of, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mnmx, static_cast<unsigned long long>(mn) ^ 0x8000000000000000ull);
    atomicMax(mnmx + 1, static_cast<unsigned long long>(mx) ^ 0x8000000000000000ull);
    if (of) atomicOr(overflow, 1);
  }
}

// ---- per-query code tables ----------------------------------------------------

struct DimFilter {
  const int32_t* col;
  int kind;
  int64_t lo, hi;
  const int64_t* set;
  int set_len;
};

struct DimGroup {
  const int32_t* col;
  int64_t mn;
  int64_t stride;
};

struct CodeArgs {
  int64_t rows;
  const int32_t* row_slot;
  int32_t* code;
  int n_filters;
  DimFilter f[kMaxDimFilters];
  int n_groups;
  DimGroup g[kMaxDimGroups];
};

__device__ __forceinline__ bool pred_eval(int kind, int64_t v, int64_t lo, int64_t hi, const int64_t* set, int n) {
  switch (kind) {  // predicate.hpp:84-93
    case LAQ_PRED_LT: return v < lo;
    case LAQ_PRED_LE: return v <= lo;
    case LAQ_PRED_EQ: return v == lo;
    case LAQ_PRED_GE: return v >= lo;
    case LAQ_PRED_GT: return v > lo;
    case LAQ_PRED_BETWEEN: return v >= lo && v <= hi;
    default: {  // InSet: binary search over the sorted set
      int a = 0, b = n;
      while (a < b) {
        const int m = (a + b) >> 1;
        const int64_t s = set[m];
        if (s == v) return true;
        if (s < v) a = m + 1; else b = m;
      }
      return false;
    }
  }
}

__global__ void code_kernel(const CodeArgs a) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < a.rows; r += (int64_t)gridDim.x * blockDim.x) {
    bool pass = true;
    for (int i = 0; i < a.n_filters && pass; ++i)
      pass = pred_eval(a.f[i].kind, a.f[i].col[r], a.f[i].lo, a.f[i].hi, a.f[i].set, a.f[i].set_len);
    int64_t code = -1;
    if (pass) {
      code = 0;
      for (int i = 0; i < a.n_groups; ++i) code += (static_cast<int64_t>(a.g[i].col[r]) - a.g[i].mn) * a.g[i].stride;
    }
    a.code[a.row_slot[r]] = static_cast<int32_t>(code);
  }
}

// ---- the fused scan --------------------------------------------------------------

struct LinkProbe {
  int kind;
  int64_t base, size;
  const int64_t* keys;
  const int32_t* code;  // per slot
};

struct FactFilter {
  const int32_t* col;
  int kind;
  int64_t lo, hi;
  const int64_t* set;
  int set_len;
};

struct FactGroup {
  const int32_t* col;
  int64_t mn, stride;
};

struct ScanArgs {
  int64_t n;
  const int32_t* fk[kMaxLinks];
  LinkProbe link[kMaxLinks];
  FactFilter ff[kMaxFactFilters];
  int n_fgroups;
  FactGroup fg[kMaxFactGroups];
  const int32_t* measure;  // nullptr: count only
  int64_t n_groups;
  unsigned long long* acc;  // [2*G]: count, sum
};

__device__ __forceinline__ int32_t link_code(const LinkProbe& p, int32_t key) {
  if (p.kind == PROBE_DIRECT) {
    const uint64_t s = static_cast<uint64_t>(static_cast<int64_t>(key) - p.base);
    return s < static_cast<uint64_t>(p.size) ? __ldg(p.code + s) : -1;
  }
  const uint64_t mask = static_cast<uint64_t>(p.size) - 1;
  uint64_t h = static_cast<uint64_t>(static_cast<int64_t>(key)) * 0x9E3779B97F4A7C15ull;
  h ^= h >> 29;
  for (uint64_t s = h & mask;; s = (s + 1) & mask) {
    const int64_t k = __ldg(p.keys + s);
    if (k == key) return __ldg(p.code + s);
    if (k < 0) return -1;
  }
}

__device__ __forceinline__ int4 ld4(const int32_t* p, int64_t row0, int64_t n, bool vec) {
  if (vec && row0 + 4 <= n) return __ldcs(reinterpret_cast<const int4*>(p + row0));
  int4 v;
  v.x = row0 + 0 < n ? p[row0 + 0] : 0;
  v.y = row0 + 1 < n ? p[row0 + 1] : 0;
  v.z = row0 + 2 < n ? p[row0 + 2] : 0;
  v.w = row0 + 3 < n ? p[row0 + 3] : 0;
  return v;
}

__device__ __forceinline__ int comp(const int4& v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }

// mode: 0 = single group held in registers, 1 = shared-memory bins, 2 = global atomics
template <int NL, int NF, int MODE>
__global__ void __launch_bounds__(kScanBlock) scan_kernel(const ScanArgs a, const bool vec) {
  extern __shared__ unsigned long long s_bins[];  // MODE 1: [G] counts then [G] sums
  if constexpr (MODE == 1) {
    for (int64_t g = threadIdx.x; g < 2 * a.n_groups; g += blockDim.x) s_bins[g] = 0;
    __syncthreads();
  }
  unsigned long long r_cnt = 0, r_sum = 0;

  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t row0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4; row0 < a.n; row0 += stride) {
    // Issue every streamed column load up front (memory-level parallelism).
    int4 fk[NL > 0 ? NL : 1], fv[NF > 0 ? NF : 1], mv;
#pragma unroll
    for (int j = 0; j < NL; ++j) fk[j] = ld4(a.fk[j], row0, a.n, vec);
#pragma unroll
    for (int f = 0; f < NF; ++f) fv[f] = ld4(a.ff[f].col, row0, a.n, vec);
    if (a.measure) mv = ld4(a.measure, row0, a.n, vec);

    int64_t gid[4];
    bool alive[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      alive[i] = row0 + i < a.n;
      gid[i] = 0;
    }
#pragma unroll
    for (int f = 0; f < NF; ++f)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        alive[i] = alive[i] && pred_eval(a.ff[f].kind, comp(fv[f], i), a.ff[f].lo, a.ff[f].hi, a.ff[f].set,
                                         a.ff[f].set_len);
#pragma unroll
    for (int j = 0; j < NL; ++j)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (alive[i]) {
          const int32_t c = link_code(a.link[j], comp(fk[j], i));
          alive[i] = c >= 0;
          gid[i] += c;
        }
    for (int g = 0; g < a.n_fgroups; ++g) {
      const int4 v = ld4(a.fg[g].col, row0, a.n, vec);
#pragma unroll
      for (int i = 0; i < 4; ++i) gid[i] += (static_cast<int64_t>(comp(v, i)) - a.fg[g].mn) * a.fg[g].stride;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (!alive[i]) continue;
      const unsigned long long val = a.measure ? static_cast<unsigned long long>(static_cast<long long>(comp(mv, i))) : 0ull;
      if constexpr (MODE == 0) {
        r_cnt += 1;
        r_sum += val;
      } else if constexpr (MODE == 1) {
        atomicAdd(s_bins + gid[i], 1ull);
        if (a.measure) atomicAdd(s_bins + a.n_groups + gid[i], val);
      } else {
        atomicAdd(a.acc + 2 * gid[i], 1ull);
        if (a.measure) atomicAdd(a.acc + 2 * gid[i] + 1, val);
      }
    }
  }

  if constexpr (MODE == 0) {
    for (int o = 16; o; o >>= 1) {
      r_cnt += __shfl_xor_sync(0xffffffffu, r_cnt, o);
      r_sum += __shfl_xor_sync(0xffffffffu, r_sum, o);
    }
    __shared__ unsigned long long w_cnt[kScanBlock / 32], w_sum[kScanBlock / 32];
    if ((threadIdx.x & 31) == 0) {
      w_cnt[threadIdx.x >> 5] = r_cnt;
      w_sum[threadIdx.x >> 5] = r_sum;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long c = 0, s = 0;
      for (int w = 0; w < kScanBlock / 32; ++w) {
        c += w_cnt[w];
        s += w_sum[w];
      }
      if (c) {
        atomicAdd(a.acc, c);
        atomicAdd(a.acc + 1, s);
      }
    }
  } else if constexpr (MODE == 1) {
    __syncthreads();
    for (int64_t g = threadIdx.x; g < a.n_groups; g += blockDim.x) {
      const unsigned long long c = s_bins[g];
      if (c) {
        atomicAdd(a.acc + 2 * g, c);
        atomicAdd(a.acc + 2 * g + 1, s_bins[a.n_groups + g]);
      }
    }
  }
}

template <int NL, int NF>
void launch_scan_nf(laq_ctx* ctx, const ScanArgs& a, bool vec, int mode, int grid) {
  const size_t smem = mode == 1 ? static_cast<size_t>(2 * a.n_groups) * sizeof(unsigned long long) : 0;
  if (mode == 0) scan_kernel<NL, NF, 0><<<grid, kScanBlock, 0, ctx->stream>>>(a, vec);
  else if (mode == 1) {
    static bool attr_set = false;  // per instantiation
    if (!attr_set) {
      LAQ_CUDA(cudaFuncSetAttribute(scan_kernel<NL, NF, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(2 * kSmemBins * sizeof(unsigned long long))));
      attr_set = true;
    }
    scan_kernel<NL, NF, 1><<<grid, kScanBlock, smem, ctx->stream>>>(a, vec);
  } else scan_kernel<NL, NF, 2><<<grid, kScanBlock, 0, ctx->stream>>>(a, vec);
}

template <int NL>
void launch_scan_nl(laq_ctx* ctx, const ScanArgs& a, int nf, bool vec, int mode, int grid) {
  switch (nf) {
    case 0: launch_scan_nf<NL, 0>(ctx, a, vec, mode, grid); break;
    case 1: launch_scan_nf<NL, 1>(ctx, a, vec, mode, grid); break;
    case 2: launch_scan_nf<NL, 2>(ctx, a, vec, mode, grid); break;
    case 3: launch_scan_nf<NL, 3>(ctx, a, vec, mode, grid); break;
    case 4: launch_scan_nf<NL, 4>(ctx, a, vec, mode, grid); break;
    default: fail(LAQ_ERR_UNSUPPORTED, "at most 4 fact filters per query");
  }
}

void launch_scan(laq_ctx* ctx, const ScanArgs& a, int nl, int nf, bool vec, int mode, int grid) {
  switch (nl) {
    case 0: launch_scan_nl<0>(ctx, a, nf, vec, mode, grid); break;
    case 1: launch_scan_nl<1>(ctx, a, nf, vec, mode, grid); break;
    case 2: launch_scan_nl<2>(ctx, a, nf, vec, mode, grid); break;
    case 3: launch_scan_nl<3>(ctx, a, nf, vec, mode, grid); break;
    case 4: launch_scan_nl<4>(ctx, a, nf, vec, mode, grid); break;
    case 5: launch_scan_nl<5>(ctx, a, nf, vec, mode, grid); break;
    case 6: launch_scan_nl<6>(ctx, a, nf, vec, mode, grid); break;
    case 7: launch_scan_nl<7>(ctx, a, nf, vec, mode, grid); break;
    case 8: launch_scan_nl<8>(ctx, a, nf, vec, mode, grid); break;
    default: fail(LAQ_ERR_UNSUPPORTED, "at most 8 joins per query");
  }
  launched(ctx);
}

}  // namespace
}  // namespace laq

using namespace laq;

struct laq_star {
  laq_ctx* ctx = nullptr;
  std::vector<std::unique_ptr<DevTable>> tables;
  int fact = -1;
  struct Link {
    std::string fk, dim, pk;
  };
  std::vector<Link> links;
  std::map<std::string, std::unique_ptr<Probe>> probes;  // "dim/pk" -> probe

  const DevTable* table(const std::string& n) const {
    for (const auto& t : tables)
      if (t->name == n) return t.get();
    return nullptr;
  }
  const DevTable* dim(const std::string& n) const {  // StarSchema::dim (storage.cpp:216-221)
    for (size_t i = 0; i < tables.size(); ++i)
      if (static_cast<int>(i) != fact && tables[i]->name == n) return tables[i].get();
    fail(LAQ_ERR_NAME, "unknown dimension: " + n);
  }
  const Probe& probe(const DevTable& d, const DevCol& pk) {
    const std::string key = d.name + "/" + pk.name;
    auto it = probes.find(key);
    if (it != probes.end()) return *it->second;
    auto p = std::make_unique<Probe>();
    build_probe(ctx, nullptr, pk.d, d.rows, *p, "multiway_star_join: duplicate keys in " + pk.name);
    return *probes.emplace(key, std::move(p)).first->second;
  }
};

namespace laq {
namespace {

const DevCol& int_col(const DevTable& t, const std::string& name) {
  const DevCol* c = t.find(name);
  if (!c) fail(LAQ_ERR_NAME, "unknown column: " + name);  // Schema::index_of, storage.cpp:25-29
  if (c->kind == LAQ_COL_FLOAT) fail(LAQ_ERR_TYPE, "table: column '" + name + "' is not integer");
  return *c;
}

void check_pred_type(const DevCol& c, const laq_filter_desc& f) {
  // predicate.hpp:95-103: typed constants vs column kind.
  const bool col_float = c.kind == LAQ_COL_FLOAT;
  if (!f.is_float && col_float) fail(LAQ_ERR_TYPE, "predicate constant is integer, column is float");
  if (f.is_float && !col_float) fail(LAQ_ERR_TYPE, "predicate constant is float, column is integer");
  if (f.is_float) fail(LAQ_ERR_UNSUPPORTED, "float predicates are not on the device path");
}

}  // namespace
}  // namespace laq

struct laq_plan {
  laq_ctx* ctx = nullptr;
  int64_t G = 1;
  int64_t fact_rows = 0;
  bool plain_sum = false;
  bool count_only = false;
  // emission: group columns in group_by order
  struct GCol {
    int64_t mn, range, stride;
  };
  std::vector<GCol> gcols;
  // per link code tables
  struct LinkCode {
    CodeArgs args;
    DevMem<int32_t> code;
    int64_t slots;
  };
  std::vector<LinkCode> links;
  DevMem<int64_t> sets;  // INSET values of every filter
  ScanArgs scan{};
  int nl = 0, nf = 0;
  bool vec = true;
  int mode = 0;
  int grid = 1;
};

extern "C" {

int laq_star_create(laq_ctx* ctx, laq_star** out) {
  return guard(ctx, [&] {
    auto* s = new laq_star();
    s->ctx = ctx;
    *out = s;
  });
}

int laq_star_destroy(laq_star* s) {
  delete s;
  return LAQ_OK;
}

static DevTable& new_table(laq_star* s, const char* name, int32_t is_fact, int64_t rows) {
  if (s->table(name)) fail(LAQ_ERR_NAME, std::string("duplicate table name: ") + name);
  if (is_fact && s->fact >= 0) fail(LAQ_ERR_SHAPE, "star schema already has a fact table");
  s->tables.push_back(std::make_unique<DevTable>());
  DevTable& t = *s->tables.back();
  t.name = name;
  t.rows = rows;
  if (is_fact) s->fact = static_cast<int>(s->tables.size()) - 1;
  return t;
}

int laq_star_add_table(laq_star* s, const char* name, int32_t is_fact, int64_t rows, int32_t n_cols,
                       const char* const* col_names, const int32_t* col_kinds, int32_t int_width,
                       const void* const* h_cols) {
  laq_ctx* ctx = s->ctx;
  return guard(ctx, [&] {
    if (int_width != 4 && int_width != 8) fail(LAQ_ERR_SHAPE, "int_width must be 4 or 8");
    if (n_cols < 1) fail(LAQ_ERR_FORMAT, "schema has no columns");
    DevTable& t = new_table(s, name, is_fact, rows);
    const int64_t chunk = std::min<int64_t>(rows, int64_t{1} << 25);
    DevMem<int64_t> stage(int_width == 8 ? static_cast<size_t>(std::max<int64_t>(chunk, 1)) : 0);
    unsigned long long* mnmx = reinterpret_cast<unsigned long long*>(ctx->d_flags + 24);
    int* overflow = reinterpret_cast<int*>(ctx->d_flags + 26);
    for (int c = 0; c < n_cols; ++c) {
      DevCol col;
      col.name = col_names[c];
      col.kind = col_kinds[c];
      for (const auto& o : t.cols)
        if (o.name == col.name) fail(LAQ_ERR_NAME, "duplicate column name: " + col.name);
      if (col.kind == LAQ_COL_FLOAT) {  // kept on the host side only (no float device path)
        t.cols.push_back(col);
        continue;
      }
      t.owned.emplace_back(static_cast<size_t>(std::max<int64_t>(rows, 1)));
      col.d = t.owned.back().get();
      if (rows > 0) {
        if (int_width == 8) {
          unsigned long long init[2] = {~0ull, 0ull};
          LAQ_CUDA(cudaMemcpyAsync(mnmx, init, sizeof init, cudaMemcpyHostToDevice, ctx->stream));
          LAQ_CUDA(cudaMemsetAsync(overflow, 0, sizeof(int), ctx->stream));
          const int64_t* src = static_cast<const int64_t*>(h_cols[c]);
          for (int64_t b = 0; b < rows; b += chunk) {
            const int64_t m = std::min(chunk, rows - b);
            LAQ_CUDA(cudaMemcpyAsync(stage.get(), src + b, m * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
            narrow_kernel<<<grid_for(m, 256 * 8, ctx->sm_count * 8), 256, 0, ctx->stream>>>(stage.get(), col.d + b, m,
                                                                                           mnmx, overflow);
            launched(ctx);
            sync(ctx);
          }
          LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, mnmx, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
          sync(ctx);
          col.mn = static_cast<int64_t>(static_cast<unsigned long long>(ctx->h_pinned[0]) ^ 0x8000000000000000ull);
          col.mx = static_cast<int64_t>(static_cast<unsigned long long>(ctx->h_pinned[1]) ^ 0x8000000000000000ull);
          if (*reinterpret_cast<int*>(ctx->h_pinned + 2))
            fail(LAQ_ERR_CAPACITY, "column '" + col.name + "' has values outside int32 (device layout)");
        } else {
          LAQ_CUDA(cudaMemcpyAsync(col.d, h_cols[c], rows * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
          minmax_i32(ctx, col.d, rows, &col.mn, &col.mx);
        }
        if (col.kind == LAQ_COL_KEY && col.mn < 0)
          fail(LAQ_ERR_FORMAT, "table: negative key in column '" + col.name + "'");
      }
      t.cols.push_back(col);
    }
  });
}

int laq_star_add_table_device(laq_star* s, const char* name, int32_t is_fact, int64_t rows, int32_t n_cols,
                              const char* const* col_names, const int32_t* col_kinds, const int32_t* const* d_cols) {
  laq_ctx* ctx = s->ctx;
  return guard(ctx, [&] {
    DevTable& t = new_table(s, name, is_fact, rows);
    for (int c = 0; c < n_cols; ++c) {
      DevCol col;
      col.name = col_names[c];
      col.kind = col_kinds[c];
      col.d = const_cast<int32_t*>(d_cols[c]);
      if (col.kind != LAQ_COL_FLOAT && rows > 0) minmax_i32(ctx, col.d, rows, &col.mn, &col.mx);
      if (col.kind == LAQ_COL_KEY && col.mn < 0)
        fail(LAQ_ERR_FORMAT, "table: negative key in column '" + col.name + "'");
      t.cols.push_back(col);
    }
  });
}

int laq_star_add_link(laq_star* s, const char* fact_fk, const char* dim_name, const char* dim_pk) {
  laq_ctx* ctx = s->ctx;
  return guard(ctx, [&] {
    // StarSchema ctor (storage.cpp:200-214): every link resolves, pks unique.
    if (s->fact < 0) fail(LAQ_ERR_SHAPE, "star schema has no fact table");
    int_col(*s->tables[s->fact], fact_fk);
    const DevTable* d = s->dim(dim_name);
    const DevCol& pk = int_col(*d, dim_pk);
    s->probe(*d, pk);
    s->links.push_back({fact_fk, dim_name, dim_pk});
  });
}

int laq_query_prepare(laq_ctx* ctx, const laq_star* cs, const laq_query_desc* q, laq_plan** out,
                      int64_t* h_n_groups) {
  laq_star* s = const_cast<laq_star*>(cs);
  return guard(ctx, [&] {
    if (s->fact < 0) fail(LAQ_ERR_SHAPE, "star schema has no fact table");
    const DevTable& fact = *s->tables[s->fact];
    auto plan = std::make_unique<laq_plan>();
    plan->ctx = ctx;
    plan->fact_rows = fact.rows;
    if (q->n_joins > kMaxLinks) fail(LAQ_ERR_UNSUPPORTED, "at most 8 joins per query");

    // Collect all INSET constants into one device array.
    std::vector<int64_t> sets;
    std::vector<int64_t> set_off(q->n_filters, 0);
    for (int i = 0; i < q->n_filters; ++i) {
      const laq_filter_desc& f = q->filters[i];
      if (f.target < -1 || f.target >= q->n_joins) fail(LAQ_ERR_INDEX, "filter target out of range");
      set_off[i] = static_cast<int64_t>(sets.size());
      if (f.kind == LAQ_PRED_INSET) {
        std::vector<int64_t> v(f.set, f.set + f.set_len);
        std::sort(v.begin(), v.end());  // Predicate::in_set sorts (predicate.hpp:69-74)
        sets.insert(sets.end(), v.begin(), v.end());
      }
    }
    plan->sets = DevMem<int64_t>(std::max<size_t>(sets.size(), 1));
    if (!sets.empty())
      LAQ_CUDA(cudaMemcpy(plan->sets.get(), sets.data(), sets.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    const int64_t* dsets = plan->sets.get();

    // Group columns: value range per column; strides mixed radix, last fastest.
    const int ng = q->n_group;
    std::vector<const DevCol*> gc(ng);
    for (int g = 0; g < ng; ++g) {
      const laq_group_desc& gd = q->group_by[g];
      if (gd.target < -1 || gd.target >= q->n_joins) fail(LAQ_ERR_INDEX, "group target out of range");
      const DevTable& t = gd.target < 0 ? fact : *s->dim(q->joins[gd.target].dim_name);
      gc[g] = &int_col(t, gd.column);
    }
    plan->gcols.resize(ng);
    int64_t G = 1;
    for (int g = ng - 1; g >= 0; --g) {
      const int64_t range = gc[g]->mx >= gc[g]->mn ? gc[g]->mx - gc[g]->mn + 1 : 1;
      plan->gcols[g] = {gc[g]->mn, range, G};
      if (range > (int64_t{1} << 30) || G > (int64_t{1} << 30) / range)
        fail(LAQ_ERR_UNSUPPORTED, "group-id space exceeds 2^30 (sort-based group-by is not on this path)");
      G *= range;
    }
    plan->G = G;
    plan->plain_sum = ng == 0;

    ScanArgs& a = plan->scan;
    a.n = fact.rows;
    a.n_groups = G;
    bool aligned = true;
    auto note_align = [&](const int32_t* p) { aligned = aligned && (reinterpret_cast<uintptr_t>(p) % 16 == 0); };
    // Measure (cli.cpp:100-101); NULL = count survivors only.
    if (q->measure) {
      const DevCol& mcol = int_col(fact, q->measure);
      a.measure = mcol.d;
      note_align(mcol.d);
    } else {
      a.measure = nullptr;
      plan->count_only = true;
    }

    // Fact filters.
    int nf = 0;
    for (int i = 0; i < q->n_filters; ++i) {
      const laq_filter_desc& f = q->filters[i];
      if (f.target != -1) continue;
      const DevCol* c = fact.find(f.column);
      if (!c) fail(LAQ_ERR_NAME, std::string("unknown column: ") + f.column);
      check_pred_type(*c, f);
      if (nf >= kMaxFactFilters) fail(LAQ_ERR_UNSUPPORTED, "at most 4 fact filters per query");
      a.ff[nf++] = FactFilter{c->d, f.kind, f.lo, f.hi, dsets + set_off[i], static_cast<int>(f.set_len)};
      note_align(c->d);
    }
    plan->nf = nf;

    // Fact group columns.
    for (int g = 0; g < ng; ++g) {
      if (q->group_by[g].target != -1) continue;
      if (a.n_fgroups >= kMaxFactGroups) fail(LAQ_ERR_UNSUPPORTED, "at most 4 fact group columns");
      a.fg[a.n_fgroups++] = FactGroup{gc[g]->d, plan->gcols[g].mn, plan->gcols[g].stride};
      note_align(gc[g]->d);
    }

    // Links: probe (cached per dim/pk) + per-query code table.
    plan->links.resize(q->n_joins);
    for (int j = 0; j < q->n_joins; ++j) {
      const laq_link_desc& l = q->joins[j];
      const DevCol& fk = int_col(fact, l.fact_fk);
      const DevTable* d = s->dim(l.dim_name);
      const DevCol& pk = int_col(*d, l.dim_pk);
      const Probe& pr = s->probe(*d, pk);
      auto& lc = plan->links[j];
      lc.slots = std::max<int64_t>(pr.size, 1);
      lc.code = DevMem<int32_t>(lc.slots);
      CodeArgs& ca = lc.args;
      ca.rows = d->rows;
      ca.row_slot = pr.row_slot.get();
      ca.code = lc.code.get();
      for (int i = 0; i < q->n_filters; ++i) {
        const laq_filter_desc& f = q->filters[i];
        if (f.target != j) continue;
        const DevCol* c = d->find(f.column);
        if (!c) fail(LAQ_ERR_NAME, std::string("unknown column: ") + f.column);
        check_pred_type(*c, f);
        if (ca.n_filters >= kMaxDimFilters) fail(LAQ_ERR_UNSUPPORTED, "at most 8 filters per dimension");
        ca.f[ca.n_filters++] = DimFilter{c->d, f.kind, f.lo, f.hi, dsets + set_off[i], static_cast<int>(f.set_len)};
      }
      for (int g = 0; g < ng; ++g) {
        if (q->group_by[g].target != j) continue;
        if (ca.n_groups >= kMaxDimGroups) fail(LAQ_ERR_UNSUPPORTED, "at most 4 group columns per dimension");
        ca.g[ca.n_groups++] = DimGroup{gc[g]->d, plan->gcols[g].mn, plan->gcols[g].stride};
      }
      a.fk[j] = fk.d;
      a.link[j] = LinkProbe{pr.kind, pr.base, pr.size, pr.keys.get(), lc.code.get()};
      note_align(fk.d);
    }
    plan->nl = q->n_joins;
    plan->vec = aligned;
    plan->mode = G == 1 ? 0 : (G <= kSmemBins ? 1 : 2);
    // Persistent grid: enough resident blocks to cover every SM several times.
    const int per_sm = plan->mode == 1 && G > 1024 ? 2 : 6;
    plan->grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ctx->sm_count * per_sm, (fact.rows + 1023) / 1024)));
    *h_n_groups = G;
    *out = plan.release();
  });
}

int laq_plan_build_codes(laq_ctx* ctx, laq_plan* p) {
  return guard(ctx, [&] {
    for (auto& lc : p->links) {
      LAQ_CUDA(cudaMemsetAsync(lc.code.get(), 0xFF, lc.slots * sizeof(int32_t), ctx->stream));
      if (lc.args.rows > 0) {
        code_kernel<<<grid_for(lc.args.rows, 256, ctx->sm_count * 8), 256, 0, ctx->stream>>>(lc.args);
        launched(ctx);
      }
    }
  });
}

int laq_plan_scan(laq_ctx* ctx, laq_plan* p, int64_t* d_acc, int32_t accumulate) {
  return guard(ctx, [&] {
    if (!accumulate) LAQ_CUDA(cudaMemsetAsync(d_acc, 0, 2 * p->G * sizeof(int64_t), ctx->stream));
    if (p->fact_rows == 0) return;
    ScanArgs a = p->scan;
    a.acc = reinterpret_cast<unsigned long long*>(d_acc);
    launch_scan(ctx, a, p->nl, p->nf, p->vec, p->mode, p->grid);
  });
}

int laq_plan_execute(laq_ctx* ctx, laq_plan* p, int64_t* d_acc, int32_t accumulate) {
  const int rc = laq_plan_build_codes(ctx, p);
  return rc ? rc : laq_plan_scan(ctx, p, d_acc, accumulate);
}

int64_t laq_plan_bytes_per_row(const laq_plan* p) {
  // fks + fact filter columns + fact group columns + measure, int32 each.
  return 4 * (p->nl + p->nf + p->scan.n_fgroups + (p->scan.measure ? 1 : 0));
}

int laq_plan_emit(const laq_plan* p, const int64_t* acc, double* out, int64_t cap, int64_t* rows, int64_t* cols) {
  try {
    const int ng = static_cast<int>(p->gcols.size());
    if (p->plain_sum) {  // dense_matmul(ones, vals): 1x1 (cli.cpp:103-107)
      *rows = 1;
      *cols = 1;
      if (cap < 1) return LAQ_ERR_CAPACITY;
      out[0] = static_cast<double>(acc[1]);
      return LAQ_OK;
    }
    int64_t r = 0;
    for (int64_t g = 0; g < p->G; ++g)
      if (acc[2 * g] != 0) ++r;
    *rows = r;
    *cols = ng + 1;
    if (r * (ng + 1) > cap) return LAQ_ERR_CAPACITY;
    int64_t o = 0;
    for (int64_t g = 0; g < p->G; ++g) {
      if (acc[2 * g] == 0) continue;  // present groups only (laqops.cpp:431-453)
      for (int c = 0; c < ng; ++c) {
        const auto& gc = p->gcols[c];
        out[o++] = static_cast<double>((g / gc.stride) % gc.range + gc.mn);
      }
      out[o++] = static_cast<double>(acc[2 * g + 1]);
    }
    return LAQ_OK;
  } catch (...) {
    return LAQ_ERR_GENERIC;
  }
}

int laq_plan_destroy(laq_plan* p) {
  delete p;
  return LAQ_OK;
}

int laq_run_query(laq_ctx* ctx, const laq_star* s, const laq_query_desc* q, double* out, int64_t cap, int64_t* rows,
                  int64_t* cols) {
  laq_plan* p = nullptr;
  int64_t G = 0;
  int rc = laq_query_prepare(ctx, s, q, &p, &G);
  if (rc) return rc;
  rc = guard(ctx, [&] {
    DevBuf<int64_t> acc(ctx, 2 * G);
    const int rc2 = laq_plan_execute(ctx, p, acc.get(), 0);
    if (rc2) fail(rc2, ctx->err);
    std::vector<int64_t> h(2 * G);
    LAQ_CUDA(cudaMemcpyAsync(h.data(), acc.get(), 2 * G * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    const int rc3 = laq_plan_emit(p, h.data(), out, cap, rows, cols);
    if (rc3) fail(rc3, "output capacity");
  });
  laq_plan_destroy(p);
  return rc;
}

int laq_measure_selectivity(laq_ctx* ctx, const laq_star* s, const laq_query_desc* q, double* out) {
  // Count survivors only: drop group-by and measure (benchgen.cpp:366-411).
  laq_query_desc c = *q;
  c.n_group = 0;
  c.measure = nullptr;
  laq_plan* p = nullptr;
  int64_t G = 0;
  int rc = laq_query_prepare(ctx, s, &c, &p, &G);
  if (rc) return rc;
  rc = guard(ctx, [&] {
    const int rc2 = laq_plan_execute(ctx, p, ctx->d_flags + 32, 0);
    if (rc2) fail(rc2, ctx->err);
    LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, ctx->d_flags + 32, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    *out = p->fact_rows == 0 ? 0.0 : static_cast<double>(ctx->h_pinned[0]) / static_cast<double>(p->fact_rows);
  });
  laq_plan_destroy(p);
  return rc;
}

}  // extern "C"
