// K4 ssb_scan_groupby host side: the query plan driver run_query_laq
// (cli.cpp:73-138) as ONE fused pass over the fact table per query.
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
//  * the scan (ssb_scan.cuh) streams the touched int32 fact columns once
//    (16-20 B/row), evaluates fact filters, probes each link, and accumulates
//    per group id an exact int64 (count, sum) into the caller's accumulator
//    (the NCCL all-reduce buffer when the fact table is sharded across GPUs).
// Integer sums are exact, so results equal the reference bit for bit.
#include <algorithm>
#include <cstdio>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "ssb_launch.cuh"
#include "ssb_shared.cuh"
#include "ssb_batch.cuh"

namespace laq {
namespace {

using scan::FactFilter;
using scan::FactGroup;
using scan::LinkProbe;
using scan::ScanArgs;
using scan::kMaxFactFilters;
using scan::kMaxFactGroups;
using scan::kMaxLinks;

constexpr int kMaxDimFilters = 8;
constexpr int kMaxDimGroups = 4;
constexpr int64_t kSmemBinsPipe = 4096;  // group ids binned in shared memory (pipe kernel)
constexpr int64_t kSmemBinsLdg = 6144;
constexpr int64_t kSmemTabMaxSlots = 49152;

struct DevCol {
  std::string name;
  int kind = LAQ_COL_INT;
  int32_t* d = nullptr;  // int32 device column (nullptr for float columns)
  int64_t mn = 0, mx = -1;
  bool padded = false;   // allocation has >= 16 readable bytes past the end
  // byte-packed copy (fact columns with a narrow range): value = stored + poff
  void* pk = nullptr;
  int pw = 4;        // 0: bit-packed (pbits per row)
  int32_t poff = 0;
  int pbits = 0;

  scan::Col view() const {  // what the stream kernel reads
    return pk ? scan::Col{pk, pw, poff, pbits} : scan::Col{d, 4, 0, 0};
  }
};

struct DevTable {
  std::string name;
  int64_t rows = 0;
  std::vector<DevCol> cols;
  // stream-ordered pool memory: a star rebuilt per call (the drop-in's
  // uncached path, the bench's e2e step) reuses its HBM without cudaMalloc
  std::vector<DevBuf<int32_t>> owned;
  std::vector<DevBuf<uint8_t>> packed_owned;

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

// min/max of a packed column's stored values (value = stored + offset).
template <class T>
__global__ void packed_minmax_kernel(const T* __restrict__ p, int64_t n, unsigned int* mnmx) {
  unsigned int mn = 0xffffffffu, mx = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned int v = p[i];
    mn = v < mn ? v : mn;
    mx = v > mx ? v : mx;
  }
  for (int o = 16; o; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mnmx, mn);
    atomicMax(mnmx + 1, mx);
  }
}

__device__ __forceinline__ int32_t col_value(const scan::Col& c, int64_t i) {
  if (c.w == 0) {  // bit-packed: row i at bit (i & 31) * bits of group i >> 5
    const uint32_t* g = static_cast<const uint32_t*>(c.p) + (i >> 5) * c.bits;
    const int bit = static_cast<int>(i & 31) * c.bits;
    const uint32_t lo = g[bit >> 5];
    const uint32_t hi = (bit & 31) + c.bits > 32 ? g[(bit >> 5) + 1] : 0u;
    const uint32_t v = __funnelshift_r(lo, hi, bit & 31);
    return static_cast<int32_t>(v & (c.bits >= 32 ? 0xffffffffu : ((1u << c.bits) - 1u))) + c.off;
  }
  if (c.w == 1) return static_cast<int32_t>(static_cast<const uint8_t*>(c.p)[i]) + c.off;
  if (c.w == 2) return static_cast<int32_t>(static_cast<const uint16_t*>(c.p)[i]) + c.off;
  return static_cast<const int32_t*>(c.p)[i];
}

// min/max of any column view (value = decoded + offset), as int64 keys ^ sign bit.
__global__ void view_minmax_kernel(const scan::Col c, int64_t n, unsigned long long* mnmx) {
  long long mn = LLONG_MAX, mx = LLONG_MIN;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const long long v = col_value(c, i);
    mn = v < mn ? v : mn;
    mx = v > mx ? v : mx;
  }
  for (int o = 16; o; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mnmx, static_cast<unsigned long long>(mn) ^ 0x8000000000000000ull);
    atomicMax(mnmx + 1, static_cast<unsigned long long>(mx) ^ 0x8000000000000000ull);
  }
}

template <class T>
__global__ void pack_kernel(const int32_t* __restrict__ src, int64_t n, int32_t off, T* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = static_cast<T>(src[i] - off);
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

__global__ void code_kernel(const CodeArgs a) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < a.rows; r += (int64_t)gridDim.x * blockDim.x) {
    bool pass = true;
    for (int i = 0; i < a.n_filters && pass; ++i)
      pass = scan::pred_eval(a.f[i].kind, a.f[i].col[r], a.f[i].lo, a.f[i].hi, a.f[i].set, a.f[i].set_len);
    int64_t code = -1;
    if (pass) {
      code = 0;
      for (int i = 0; i < a.n_groups; ++i) code += (static_cast<int64_t>(a.g[i].col[r]) - a.g[i].mn) * a.g[i].stride;
    }
    a.code[a.row_slot[r]] = static_cast<int32_t>(code);
  }
}

// Every link's code table of a query in one launch, one thread per probe slot:
// slot -> dim row (probe table) -> filters -> group code, -1 for an empty slot
// or a failing row.  Replaces a memset + code_kernel pair per link (bench
// step: 2 launches per query instead of 2 per link + 1).
constexpr int kMaxCodeLinks = 24;  // links per fused code launch (a batch of up to 6 SSB queries)
struct MultiCodeArgs {
  int n;
  int64_t start[kMaxCodeLinks + 1];  // prefix of slot counts, each rounded up to 32
  int64_t slots[kMaxCodeLinks];
  const int32_t* slot_row[kMaxCodeLinks];
  int fmt[kMaxCodeLinks];
  void* packed[kMaxCodeLinks];
  CodeArgs link[kMaxCodeLinks];
};

// Links start at multiples of 32 slots, so a warp's 32 consecutive indices are
// 32 consecutive slots of one link (the bitmap word is one warp ballot).
__global__ void codes_kernel(const MultiCodeArgs m) {
  const int64_t total = m.start[m.n];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int j = 0;
    while (i >= m.start[j + 1]) ++j;
    const CodeArgs& a = m.link[j];
    const int64_t s = i - m.start[j];
    const bool in = s < m.slots[j];
    const int32_t r = in && m.slot_row[j] ? __ldg(m.slot_row[j] + s) : -1;
    int64_t code = -1;
    if (r >= 0) {
      bool pass = true;
      for (int f = 0; f < a.n_filters && pass; ++f)
        pass = scan::pred_eval(a.f[f].kind, a.f[f].col[r], a.f[f].lo, a.f[f].hi, a.f[f].set, a.f[f].set_len);
      if (pass) {
        code = 0;
        for (int g = 0; g < a.n_groups; ++g) code += (static_cast<int64_t>(a.g[g].col[r]) - a.g[g].mn) * a.g[g].stride;
      }
    }
    if (in) a.code[s] = static_cast<int32_t>(code);
    const int fmt = m.fmt[j];
    if (fmt == scan::kFmtS16) {
      if (in) static_cast<int16_t*>(m.packed[j])[s] = static_cast<int16_t>(code);
    } else if (fmt == scan::kFmtU8) {
      if (in) static_cast<uint8_t*>(m.packed[j])[s] = code < 0 ? 255 : static_cast<uint8_t>(code);
    } else if (fmt == scan::kFmtBit) {
      const unsigned bits = __ballot_sync(0xffffffffu, code >= 0);
      if ((threadIdx.x & 31) == 0) static_cast<uint32_t*>(m.packed[j])[s >> 5] = bits;
    }
  }
}

__global__ void count_pass_kernel(const int32_t* __restrict__ code, int64_t slots, unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < slots; s += (int64_t)gridDim.x * blockDim.x)
    c += code[s] >= 0 ? 1 : 0;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// Fact FK values without a matching dim row (referential coverage of a link).
__global__ void fk_miss_kernel(const scan::Col fk, int64_t n, const ProbeView pv, unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c += pv.row(col_value(fk, i)) < 0 ? 1 : 0;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// ---- kernel dispatch (instantiated per link count in ssb_scan_nl*.cu) -----

void launch_scan(laq_ctx* ctx, const ScanArgs& a, int nl, int nf, int mode, int variant, bool vec, int grid,
                 size_t smem) {
  switch (nl) {
    case 0: scan::launch_nl<0>(ctx, a, nf, mode, variant, vec, grid, smem); break;
    case 1: scan::launch_nl<1>(ctx, a, nf, mode, variant, vec, grid, smem); break;
    case 2: scan::launch_nl<2>(ctx, a, nf, mode, variant, vec, grid, smem); break;
    case 3: scan::launch_nl<3>(ctx, a, nf, mode, variant, vec, grid, smem); break;
    case 4: scan::launch_nl<4>(ctx, a, nf, mode, variant, vec, grid, smem); break;
    case 5: scan::launch_nl<5>(ctx, a, nf, mode, variant, vec, grid, smem); break;
    case 6: scan::launch_nl<6>(ctx, a, nf, mode, variant, vec, grid, smem); break;
    default: fail(LAQ_ERR_UNSUPPORTED, "at most 6 joins per query");
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
  // "fk|dim/pk" -> every fact FK value has a dim row (computed once per star on
  // the device; cleared whenever a table is added)
  std::map<std::string, bool> covered;

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

// A fact predicate as a closed int32 interval (branch-free in the scan), or InSet.
FactFilter lower_filter(const int32_t* col, const laq_filter_desc& f, const int64_t* dset) {
  FactFilter r{col, 1, 0, 0, dset, static_cast<int>(f.set_len)};
  if (f.kind == LAQ_PRED_INSET) {
    r.inset = 1;
    return r;
  }
  int64_t lo = INT64_MIN, hi = INT64_MAX;
  switch (f.kind) {  // predicate.hpp:84-89 over integers
    case LAQ_PRED_LT: hi = f.lo == INT64_MIN ? INT64_MIN : f.lo - 1; if (f.lo == INT64_MIN) lo = 1; break;
    case LAQ_PRED_LE: hi = f.lo; break;
    case LAQ_PRED_EQ: lo = hi = f.lo; break;
    case LAQ_PRED_GE: lo = f.lo; break;
    case LAQ_PRED_GT: lo = f.lo == INT64_MAX ? INT64_MAX : f.lo + 1; if (f.lo == INT64_MAX) hi = 0; break;
    default: lo = f.lo; hi = f.hi; break;  // Between, inclusive
  }
  lo = std::max<int64_t>(lo, INT32_MIN);
  hi = std::min<int64_t>(hi, INT32_MAX);
  if (lo <= hi) {
    r.lo = static_cast<int32_t>(lo);
    r.hi = static_cast<int32_t>(hi);
  }  // else stays the empty interval [1, 0]
  return r;
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
  struct GCol {
    int64_t mn, range, stride;
  };
  std::vector<GCol> gcols;  // emission: group columns in group_by order
  struct LinkCode {
    CodeArgs args;
    DevMem<int32_t> code;
    int64_t slots;       // allocated (>= 1)
    int64_t slots_used;  // slots the fused code kernel writes (= slots)
    const int32_t* slot_row = nullptr;
    int64_t max_code = 0;  // largest group-id contribution of this link
    int fmt = scan::kFmtGlobal;  // compact copy for the direct scan (ssb_scan.cuh)
    DevMem<uint8_t> packed;
    int64_t packed_bytes = 0;  // multiple of 16
  };
  std::vector<LinkCode> links;  // in query join order
  DevMem<int64_t> sets;         // INSET values of every filter
  ScanArgs scan{};              // links in probe order
  int nl = 0, nf = 0;
  bool vec = true;
  bool pipe = false;
  int variant = 0;  // 0 ldg fallback, 1 TMA pipe, 2 resident-table stream, 3 stream over packed columns
  bool packed_only = false;
  int mode = 0;
  int grid = 1;
  size_t smem = 0;
  int64_t bytes_per_row = 0;
  int64_t measure_min = 0;  // smallest measure value (batched scans: presence by non-zero sum when > 0)
};

namespace laq {
namespace {

// Every link's code table of a batch of plans in one codes_kernel launch.
// Returns false (nothing launched) when the batch has more links than one
// launch carries.
bool build_codes_fused(laq_ctx* ctx, laq_plan* const* ps, int np) {
  MultiCodeArgs m{};
  int n = 0;
  for (int i = 0; i < np; ++i) n += static_cast<int>(ps[i]->links.size());
  if (n == 0) return true;
  if (n > kMaxCodeLinks) return false;
  for (int i = 0; i < np; ++i)
    for (const auto& lc : ps[i]->links) {
      m.link[m.n] = lc.args;
      m.slot_row[m.n] = lc.slot_row;
      m.slots[m.n] = lc.slots_used;
      m.fmt[m.n] = lc.fmt;
      m.packed[m.n] = lc.packed.get();
      m.start[m.n + 1] = m.start[m.n] + ((lc.slots_used + 31) & ~int64_t{31});
      ++m.n;
    }
  if (m.start[m.n] > 0) {
    codes_kernel<<<grid_for(m.start[m.n], 256, ctx->sm_count * 8), 256, 0, ctx->stream>>>(m);
    launched(ctx);
  }
  return true;
}

void build_codes(laq_ctx* ctx, laq_plan* p) {
  bool compact = false;
  for (auto& lc : p->links) compact = compact || lc.fmt != scan::kFmtGlobal;
  if ((compact || !std::getenv("LAQ_CODES_PER_LINK")) && build_codes_fused(ctx, &p, 1)) return;
  if (compact) fail(LAQ_ERR_UNSUPPORTED, "more links than one code launch carries");
  for (auto& lc : p->links) {
    LAQ_CUDA(cudaMemsetAsync(lc.code.get(), 0xFF, lc.slots * sizeof(int32_t), ctx->stream));
    if (lc.args.rows > 0) {
      code_kernel<<<grid_for(lc.args.rows, 256, ctx->sm_count * 8), 256, 0, ctx->stream>>>(lc.args);
      launched(ctx);
    }
  }
}

// Decide the scan's probe order, shared-memory layout, grid and bins.
void lay_out_scan(laq_ctx* ctx, laq_plan* p, const std::vector<const int32_t*>& fks,
                  const std::vector<scan::Col>& fkcols, const std::vector<const Probe*>& probes, int64_t measure_min, int64_t measure_max, bool all_padded) {
  ScanArgs& a = p->scan;
  const int nl = static_cast<int>(p->links.size());
  // Pass fraction of each link (dim rows surviving its filters), measured once.
  std::vector<double> frac(nl, 1.0);
  if (nl > 0) {
    build_codes(ctx, p);
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(ctx->d_flags + 56);
    for (int j = 0; j < nl; ++j) {
      LAQ_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), ctx->stream));
      count_pass_kernel<<<grid_for(p->links[j].slots, 256, ctx->sm_count * 4), 256, 0, ctx->stream>>>(
          p->links[j].code.get(), p->links[j].slots, cnt);
      launched(ctx);
      LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned + j, cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
      sync(ctx);
    }
    for (int j = 0; j < nl; ++j)
      frac[j] = p->links[j].args.rows ? static_cast<double>(ctx->h_pinned[j]) / p->links[j].args.rows : 0.0;
  }
  // Shared-memory budget of the pipelined kernel.
  int optin = 0;
  LAQ_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  const int64_t budget = static_cast<int64_t>(optin) - 2048;  // static smem + mbarriers
  const int nc = p->nl + p->nf + (a.measure ? 1 : 0);
  const int64_t stage_bytes = static_cast<int64_t>(nc) * scan::kTile * 4;
  // 32-bit bins are exact when the largest sum one CTA can add between two
  // spills fits 32 bits.  The widest step of any scan kernel is the direct
  // kernel's 1024 threads x 4 rows = 4096 rows, so vmax < 2^20 keeps even a
  // flush_every of 1 exact (4096 * vmax < 2^32); wider measures take 64-bit bins.
  const int64_t vmax = a.measure ? std::max<int64_t>(measure_max, 1) : 1;
  const bool narrow = a.measure == nullptr ||
                      (measure_min >= 0 && vmax * int64_t{scan::kDirectThreads} * 4 < (int64_t{1} << 32));
  const int64_t bin_bytes = p->mode == 1 ? (narrow ? 8 : 16) * p->G : 0;
  const int64_t tab_budget = budget - bin_bytes - 4 * stage_bytes;

  // The direct-probe kernel (ssb_scan.cuh) when every link is a DIRECT table,
  // the group id comes from the links only and the bins are narrow: every SSB
  // query.  LAQ_SCAN=stream|pipe|ldg selects the generic kernels.
  const char* want_env = std::getenv("LAQ_SCAN");
  bool inset_filter = false;
  for (int f = 0; f < p->nf; ++f) inset_filter = inset_filter || a.ff[f].inset;
  bool direct = (!want_env || std::string(want_env) == "direct") && p->vec && all_padded && !inset_filter && nc >= 1 && a.n_fgroups == 0 && p->mode != 2 &&
                (p->mode == 0 || narrow) && nl <= static_cast<int>(kMaxCodeLinks);
  for (int j = 0; j < nl; ++j) direct = direct && probes[j]->kind == PROBE_DIRECT;
  if (direct) {
    const int64_t dbins = p->mode == 1 ? 8 * p->G : 0;
    int64_t room = budget - dbins;
    // Each link's most compact shared format; smallest tables first while they fit.
    std::vector<int64_t> need(nl, 0);
    std::vector<int> fmt(nl, scan::kFmtGlobal);
    for (int j = 0; j < nl; ++j) {
      const auto& lc = p->links[j];
      // lc.slots = max(probe size, 1): an empty dimension still gets a one-slot
      // (all-fail) compact table, which codes_kernel writes.
      const int64_t slots = lc.slots;
      if (lc.args.n_groups == 0) fmt[j] = scan::kFmtBit, need[j] = ((slots + 31) / 32) * 4;
      else if (lc.max_code <= 254) fmt[j] = scan::kFmtU8, need[j] = slots;
      else if (lc.max_code <= 32767) fmt[j] = scan::kFmtS16, need[j] = 2 * slots;
      need[j] = (need[j] + 15) & ~int64_t{15};
    }
    std::vector<int> by(nl);
    std::iota(by.begin(), by.end(), 0);
    std::stable_sort(by.begin(), by.end(), [&](int x, int y) { return need[x] < need[y]; });
    std::vector<char> staged(nl, 0);
    for (int j : by) {
      if (std::getenv("LAQ_NOSMEMTAB") || fmt[j] == scan::kFmtGlobal || need[j] > room) continue;
      staged[j] = 1;
      room -= need[j];
    }
    // Second pass: a staged pass bitmap becomes a uint8 table (one LDS.U8 per
    // probe instead of shift/LDS/shift/and) when the remaining room allows;
    // upgrades never evict another link's table.
    for (int j : by) {
      if (!staged[j] || fmt[j] != scan::kFmtBit) continue;
      const int64_t u8 = (p->links[j].slots + 15) & ~int64_t{15};
      if (u8 - need[j] <= room) {
        room -= u8 - need[j];
        fmt[j] = scan::kFmtU8;
        need[j] = u8;
      }
    }
    int64_t off = 0;
    std::vector<int64_t> smem_off(nl, -1);
    for (int j : by) {
      auto& lc = p->links[j];
      lc.fmt = scan::kFmtGlobal;
      if (!staged[j]) continue;
      lc.fmt = fmt[j];
      lc.packed_bytes = need[j];
      lc.packed = DevMem<uint8_t>(need[j]);
      smem_off[j] = off;  // bytes
      off += need[j];
    }
    build_codes(ctx, p);  // fills the compact copies
    std::vector<double> rank(nl);
    for (int j = 0; j < nl; ++j) rank[j] = (p->links[j].fmt != scan::kFmtGlobal ? 1.0 : 8.0) / std::max(1.0 - frac[j], 1e-9);
    std::vector<int> order(nl);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return rank[x] < rank[y]; });
    bool gathers = false;
    for (int q = 0; q < nl; ++q) {
      const int j = order[q];
      const Probe& pr = *probes[j];
      const auto& lc = p->links[j];
      a.fk[q] = fks[j];
      a.fkc[q] = fkcols[j];
      LinkProbe lp{pr.kind, pr.base, pr.size, pr.keys.get(), lc.code.get(), -1};
      lp.fmt = lc.fmt;
      lp.smem_byte = lc.fmt != scan::kFmtGlobal ? static_cast<int>(smem_off[j]) : 0;
      lp.smem_bytes = static_cast<int>(lc.packed_bytes);
      lp.packed = lc.packed.get();
      a.link[q] = lp;
      gathers = gathers || lc.fmt == scan::kFmtGlobal;
    }
    a.smem_tab_elems = static_cast<int>(off);  // bytes for this kernel
    a.narrow_bins = narrow ? 1 : 0;
    a.flush_every = std::max<int64_t>(1, (int64_t{1} << 32) / (int64_t{scan::kDirectThreads} * 4 * vmax) - 1);
    // L2 prefetch of the fact rows 2 grid steps ahead when some link gathers
    // from L2 (Q2.x at SF=10: 0.184 -> 0.169 ms); plans probing shared memory
    // only run at the copy bandwidth and measured slower with it (0.144 -> 0.160).
    a.prefetch = gathers ? 2 : 0;
    if (const char* pf = std::getenv("LAQ_PREFETCH")) a.prefetch = std::atoi(pf);
    p->variant = 4;
    p->smem = static_cast<size_t>(off + dbins);
    p->grid = ctx->sm_count;  // one 1024-thread CTA per SM
    p->pipe = false;
    return;
  }

  // 1) Which code tables live in shared memory: smallest first while they fit.
  std::vector<int> by_size(nl);
  std::iota(by_size.begin(), by_size.end(), 0);
  std::stable_sort(by_size.begin(), by_size.end(), [&](int x, int y) { return probes[x]->size < probes[y]->size; });
  std::vector<int64_t> smem_off(nl, -1);
  int64_t tab_elems = 0;
  for (int j : by_size) {
    const Probe& pr = *probes[j];
    const int64_t need = (pr.size + 7) & ~int64_t{7};
    if (!std::getenv("LAQ_NOSMEMTAB") && pr.kind == PROBE_DIRECT && pr.size <= kSmemTabMaxSlots && p->G <= 32767 &&
        (tab_elems + need) * 2 <= tab_budget) {
      smem_off[j] = tab_elems;
      tab_elems += need;
    }
  }
  // 2) Probe order: ascending rank cost / (1 - pass fraction) (the classic
  // ordering of independent filters), cost ~ 1 smem lookup, 8 L2 gather, 16 hash.
  std::vector<double> rank(nl);
  for (int j = 0; j < nl; ++j) {
    const double cost = smem_off[j] >= 0 ? 1.0 : (probes[j]->kind == PROBE_HASH ? 16.0 : 8.0);
    rank[j] = cost / std::max(1.0 - frac[j], 1e-9);
  }
  std::vector<int> order(nl);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return rank[x] < rank[y]; });
  for (int q = 0; q < nl; ++q) {
    const int j = order[q];
    const Probe& pr = *probes[j];
    a.fk[q] = fks[j];
    a.fkc[q] = fkcols[j];
    a.link[q] = LinkProbe{pr.kind, pr.base, pr.size, pr.keys.get(), p->links[j].code.get(), static_cast<int>(smem_off[j])};
  }
  const int64_t rest = budget - bin_bytes - tab_elems * 2;
  int64_t stages = std::min<int64_t>(scan::kMaxStages, rest / std::max<int64_t>(stage_bytes, 1));
  if (const char* v = std::getenv("LAQ_STAGES")) stages = std::min<int64_t>(stages, std::atoi(v));  // diagnostics
  bool fact_inset = false;
  for (int f = 0; f < p->nf; ++f) fact_inset = fact_inset || a.ff[f].inset;
  // Variant: the resident-table stream kernel by default (fastest measured on
  // B200 for every SSB shape, profiles/), the TMA pipeline on request, the
  // plain-load kernel for unaligned / InSet / very wide group-id plans.
  const bool fast_ok = p->vec && all_padded && !fact_inset && nc >= 1 && (p->mode != 1 || p->G <= kSmemBinsPipe);
  const char* want = std::getenv("LAQ_SCAN");
  const std::string pick = p->packed_only ? std::string("stream") : (want ? std::string(want) : std::string("stream"));
  a.smem_tab_elems = static_cast<int>(tab_elems);
  a.narrow_bins = narrow ? 1 : 0;
  const size_t tab_bytes = static_cast<size_t>((tab_elems * 2 + 15) & ~15);
  if (fast_ok && pick == "pipe" && stages >= 2) {
    p->variant = 1;
    a.stages = static_cast<int>(stages);
    // u32 sums: between spills a CTA adds at most flush_every * kTile values <= vmax.
    a.flush_every = std::max<int64_t>(1, (int64_t{1} << 32) / (int64_t{scan::kTile} * vmax) - 1);
    p->smem = static_cast<size_t>(stages * stage_bytes + 16 * scan::kMaxStages) + tab_bytes + static_cast<size_t>(bin_bytes);
    const int64_t tiles = (p->fact_rows + scan::kTile - 1) / scan::kTile;
    p->grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ctx->sm_count, tiles)));
  } else if (fast_ok && pick != "ldg" && static_cast<int64_t>(tab_bytes) + bin_bytes <= budget) {
    p->variant = 2;
    a.flush_every = std::max<int64_t>(1, (int64_t{1} << 32) / (int64_t{scan::kStreamThreads} * 4 * vmax) - 1);
    p->smem = tab_bytes + static_cast<size_t>(bin_bytes);
    p->grid = ctx->sm_count;  // x resident CTAs per SM (occupancy, at launch)
  } else {
    p->variant = 0;
    for (int q = 0; q < nl; ++q) a.link[q].smem_off = -1;
    p->smem = p->mode == 1 ? static_cast<size_t>(2 * p->G) * sizeof(unsigned long long) : 0;
    const int per_sm = p->mode == 1 && p->G > 1024 ? 2 : 6;
    p->grid = static_cast<int>(
        std::max<int64_t>(1, std::min<int64_t>(ctx->sm_count * per_sm, (p->fact_rows + 1023) / 1024)));
  }
  p->pipe = p->variant == 1;
}

}  // namespace
}  // namespace laq

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
  s->covered.clear();
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
    // int64 host columns go H2D through a staging buffer in 128M-row (1 GB)
    // pieces, narrowed on the device; the pieces are stream-ordered, so the copy
    // engine runs back to back (measured pinned H2D on B200: 49 GB/s in 256 MB
    // pieces with a host sync after each, 55.6 GB/s in 1 GB pieces).
    const int64_t chunk = std::min<int64_t>(rows, int64_t{1} << 27);
    DevBuf<int64_t> stage(ctx, int_width == 8 ? static_cast<size_t>(std::max<int64_t>(chunk, 1)) : 0);
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
      // +4 elements: bulk copies of the last tile may read up to 12 bytes past the end.
      t.owned.emplace_back(ctx, static_cast<size_t>(rows + 4));
      col.d = t.owned.back().get();
      col.padded = true;
      LAQ_CUDA(cudaMemsetAsync(col.d + rows, 0, 4 * sizeof(int32_t), ctx->stream));
      if (rows > 0) {
        if (int_width == 8) {
          unsigned long long init[2] = {~0ull, 0ull};
          LAQ_CUDA(cudaMemcpyAsync(mnmx, init, sizeof init, cudaMemcpyHostToDevice, ctx->stream));
          LAQ_CUDA(cudaMemsetAsync(overflow, 0, sizeof(int), ctx->stream));
          const int64_t* src = static_cast<const int64_t*>(h_cols[c]);
          for (int64_t b = 0; b < rows; b += chunk) {
            const int64_t m = std::min(chunk, rows - b);
            LAQ_CUDA(cudaMemcpyAsync(stage.get(), src + b, m * sizeof(int64_t), cudaMemcpyDefault, ctx->stream));
            narrow_kernel<<<grid_for(m, 256 * 8, ctx->sm_count * 8), 256, 0, ctx->stream>>>(stage.get(), col.d + b, m,
                                                                                           mnmx, overflow);
            launched(ctx);
          }
          LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, mnmx, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
          sync(ctx);
          col.mn = static_cast<int64_t>(static_cast<unsigned long long>(ctx->h_pinned[0]) ^ 0x8000000000000000ull);
          col.mx = static_cast<int64_t>(static_cast<unsigned long long>(ctx->h_pinned[1]) ^ 0x8000000000000000ull);
          if (*reinterpret_cast<int*>(ctx->h_pinned + 2))
            fail(LAQ_ERR_CAPACITY, "column '" + col.name + "' has values outside int32 (device layout)");
        } else {
          LAQ_CUDA(cudaMemcpyAsync(col.d, h_cols[c], rows * sizeof(int32_t), cudaMemcpyDefault, ctx->stream));
          minmax_i32(ctx, col.d, rows, &col.mn, &col.mx);
        }
        if (col.kind == LAQ_COL_KEY && col.mn < 0)
          fail(LAQ_ERR_FORMAT, "table: negative key in column '" + col.name + "'");
        // Opt-in (LAQ_PACK=1): fact columns with a narrow value range also get a
        // byte-packed copy (1 or 2 bytes per row, relative to the minimum) for the
        // stream scan.  Measured on B200 (SF=10, 6 queries): 1.53 ms/step packed vs
        // 1.35 ms unpacked -- the int32 scan already issues at ~68 % of the slots,
        // and unpacking adds more instructions per row than the halved bytes save.
        const int64_t range = col.mx - col.mn;
        if (is_fact && range < 65536 && std::getenv("LAQ_PACK")) {
          col.pw = range < 256 ? 1 : 2;
          col.poff = static_cast<int32_t>(col.mn);
          t.packed_owned.emplace_back(ctx, static_cast<size_t>(rows * col.pw + 16));
          col.pk = t.packed_owned.back().get();
          LAQ_CUDA(cudaMemsetAsync(static_cast<uint8_t*>(col.pk) + rows * col.pw, 0, 16, ctx->stream));
          const int g = grid_for(rows, 256 * 8, ctx->sm_count * 8);
          if (col.pw == 1)
            pack_kernel<uint8_t><<<g, 256, 0, ctx->stream>>>(col.d, rows, col.poff, static_cast<uint8_t*>(col.pk));
          else
            pack_kernel<uint16_t><<<g, 256, 0, ctx->stream>>>(col.d, rows, col.poff, static_cast<uint16_t*>(col.pk));
          launched(ctx);
        }
      }
      t.cols.push_back(col);
    }
    sync(ctx);
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
      col.padded = rows % 4 == 0;  // whole 16-byte tail: no read past the end
      if (col.kind != LAQ_COL_FLOAT && rows > 0) minmax_i32(ctx, col.d, rows, &col.mn, &col.mx);
      if (col.kind == LAQ_COL_KEY && col.mn < 0)
        fail(LAQ_ERR_FORMAT, "table: negative key in column '" + col.name + "'");
      t.cols.push_back(col);
    }
  });
}

int laq_star_add_table_device_packed(laq_star* s, const char* name, int32_t is_fact, int64_t rows, int32_t n_cols,
                                     const char* const* col_names, const int32_t* col_kinds,
                                     const void* const* d_cols, const int32_t* widths, const int32_t* offsets) {
  laq_ctx* ctx = s->ctx;
  return guard(ctx, [&] {
    DevTable& t = new_table(s, name, is_fact, rows);
    unsigned int* mnmx = reinterpret_cast<unsigned int*>(ctx->d_flags + 30);
    for (int c = 0; c < n_cols; ++c) {
      DevCol col;
      col.name = col_names[c];
      col.kind = col_kinds[c];
      if (col.kind == LAQ_COL_FLOAT) {
        t.cols.push_back(col);
        continue;
      }
      const int w = widths[c];
      if (w != 1 && w != 2 && w != 4) fail(LAQ_ERR_SHAPE, "packed column width must be 1, 2 or 4");
      col.padded = true;  // caller contract: >= 16 readable bytes past the end
      if (w == 4) {
        if (offsets[c] != 0) fail(LAQ_ERR_SHAPE, "4-byte packed columns carry no offset");
        col.d = const_cast<int32_t*>(static_cast<const int32_t*>(d_cols[c]));
        if (rows > 0) minmax_i32(ctx, col.d, rows, &col.mn, &col.mx);
      } else {
        col.pk = const_cast<void*>(d_cols[c]);
        col.pw = w;
        col.poff = offsets[c];
        if (rows > 0) {
          const unsigned int init[2] = {0xffffffffu, 0u};
          LAQ_CUDA(cudaMemcpyAsync(mnmx, init, sizeof init, cudaMemcpyHostToDevice, ctx->stream));
          const int g = grid_for(rows, 256 * 8, ctx->sm_count * 8);
          if (w == 1)
            packed_minmax_kernel<uint8_t><<<g, 256, 0, ctx->stream>>>(static_cast<const uint8_t*>(col.pk), rows, mnmx);
          else
            packed_minmax_kernel<uint16_t><<<g, 256, 0, ctx->stream>>>(static_cast<const uint16_t*>(col.pk), rows, mnmx);
          launched(ctx);
          LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, mnmx, 2 * sizeof(unsigned int), cudaMemcpyDeviceToHost, ctx->stream));
          sync(ctx);
          const unsigned int* mm = reinterpret_cast<const unsigned int*>(ctx->h_pinned);
          col.mn = static_cast<int64_t>(mm[0]) + col.poff;
          col.mx = static_cast<int64_t>(mm[1]) + col.poff;
        }
      }
      if (col.kind == LAQ_COL_KEY && rows > 0 && col.mn < 0)
        fail(LAQ_ERR_FORMAT, "table: negative key in column '" + col.name + "'");
      t.cols.push_back(col);
    }
  });
}

int laq_star_add_table_device_bitpacked(laq_star* s, const char* name, int32_t is_fact, int64_t rows, int32_t n_cols,
                                        const char* const* col_names, const int32_t* col_kinds,
                                        const void* const* d_cols, const int32_t* bits, const int32_t* offsets) {
  laq_ctx* ctx = s->ctx;
  return guard(ctx, [&] {
    DevTable& t = new_table(s, name, is_fact, rows);
    unsigned long long* mnmx = reinterpret_cast<unsigned long long*>(ctx->d_flags + 32);
    for (int c = 0; c < n_cols; ++c) {
      DevCol col;
      col.name = col_names[c];
      col.kind = col_kinds[c];
      for (const auto& o : t.cols)
        if (o.name == col.name) fail(LAQ_ERR_NAME, "duplicate column name: " + col.name);
      if (col.kind == LAQ_COL_FLOAT) {
        t.cols.push_back(col);
        continue;
      }
      if (bits[c] < 1 || bits[c] > 32) fail(LAQ_ERR_SHAPE, "bit-packed column width must be 1..32 bits");
      if ((reinterpret_cast<uintptr_t>(d_cols[c]) & 3) != 0) fail(LAQ_ERR_SHAPE, "bit-packed column must be 4-byte aligned");
      col.padded = true;  // caller contract: whole 128-row blocks of words + 16 bytes
      col.pk = const_cast<void*>(d_cols[c]);
      col.pw = 0;
      col.pbits = bits[c];
      col.poff = offsets[c];
      if (rows > 0) {
        const unsigned long long init[2] = {~0ull, 0ull};
        LAQ_CUDA(cudaMemcpyAsync(mnmx, init, sizeof init, cudaMemcpyHostToDevice, ctx->stream));
        view_minmax_kernel<<<grid_for(rows, 256 * 8, ctx->sm_count * 8), 256, 0, ctx->stream>>>(col.view(), rows, mnmx);
        launched(ctx);
        LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, mnmx, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
        sync(ctx);
        col.mn = static_cast<int64_t>(static_cast<unsigned long long>(ctx->h_pinned[0]) ^ 0x8000000000000000ull);
        col.mx = static_cast<int64_t>(static_cast<unsigned long long>(ctx->h_pinned[1]) ^ 0x8000000000000000ull);
      }
      if (col.kind == LAQ_COL_KEY && rows > 0 && col.mn < 0)
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

namespace laq {
namespace {
bool link_covered(laq_ctx* ctx, laq_star* s, const DevCol& fk, const DevTable& d, const DevCol& pk, const Probe& pr) {
  if (std::getenv("LAQ_NO_LINK_ELISION")) return false;
  const std::string key = fk.name + "|" + d.name + "/" + pk.name;
  auto it = s->covered.find(key);
  if (it != s->covered.end()) return it->second;
  const int64_t n = s->tables[s->fact]->rows;
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(ctx->d_flags + 57);
  LAQ_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), ctx->stream));
  if (n > 0) {
    fk_miss_kernel<<<grid_for(n, 256, ctx->sm_count * 8), 256, 0, ctx->stream>>>(fk.view(), n, pr.view(), cnt);
    launched(ctx);
  }
  LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  const bool cov = ctx->h_pinned[0] == 0;
  s->covered[key] = cov;
  return cov;
}
}  // namespace
}  // namespace laq

int laq_query_prepare(laq_ctx* ctx, const laq_star* cs, const laq_query_desc* q, laq_plan** out,
                      int64_t* h_n_groups) {
  laq_star* s = const_cast<laq_star*>(cs);
  return guard(ctx, [&] {
    if (s->fact < 0) fail(LAQ_ERR_SHAPE, "star schema has no fact table");
    const DevTable& fact = *s->tables[s->fact];
    auto plan = std::make_unique<laq_plan>();
    plan->ctx = ctx;
    plan->fact_rows = fact.rows;
    if (q->n_joins > 6) fail(LAQ_ERR_UNSUPPORTED, "at most 6 joins per query");

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
    bool aligned = true, padded = true;
    bool packed_only = false;  // some scanned column exists only byte-packed (stream kernel only)
    auto note = [&](const DevCol& c) {
      aligned = aligned && (reinterpret_cast<uintptr_t>(c.d ? static_cast<const void*>(c.d) : c.pk) % 16 == 0);
      padded = padded && c.padded;
      packed_only = packed_only || c.d == nullptr;
    };
    // Measure (cli.cpp:100-101); NULL = count survivors only.
    int64_t mmin = 0, mmax = 0;
    if (q->measure) {
      const DevCol& mcol = int_col(fact, q->measure);
      a.measure = mcol.d ? mcol.d : static_cast<const int32_t*>(mcol.pk);  // (stream kernel: "has a measure")
      a.mc = mcol.view();
      mmin = mcol.mn;
      mmax = mcol.mx;
      note(mcol);
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
      a.ffc[nf] = c->view();
      a.ff[nf++] = lower_filter(c->d, f, dsets + set_off[i]);
      note(*c);
    }
    plan->nf = nf;

    // Fact group columns.
    for (int g = 0; g < ng; ++g) {
      if (q->group_by[g].target != -1) continue;
      if (a.n_fgroups >= kMaxFactGroups) fail(LAQ_ERR_UNSUPPORTED, "at most 4 fact group columns");
      if (!gc[g]->d) fail(LAQ_ERR_UNSUPPORTED, "group-by on a byte-packed fact column");
      a.fg[a.n_fgroups++] = FactGroup{gc[g]->d, plan->gcols[g].mn, plan->gcols[g].stride};
    }

    // Links: probe (cached per dim/pk) + per-query code table.
    plan->links.resize(q->n_joins);
    std::vector<const int32_t*> fks(q->n_joins);
    std::vector<const Probe*> probes(q->n_joins);
    std::vector<scan::Col> fkcols(q->n_joins);
    std::vector<char> elide(q->n_joins, 0);
    for (int j = 0; j < q->n_joins; ++j) {
      const laq_link_desc& l = q->joins[j];
      const DevCol& fk = int_col(fact, l.fact_fk);
      const DevTable* d = s->dim(l.dim_name);
      const DevCol& pk = int_col(*d, l.dim_pk);
      const Probe& pr = s->probe(*d, pk);
      auto& lc = plan->links[j];
      lc.slots = std::max<int64_t>(pr.size, 1);
      lc.slots_used = lc.slots;
      lc.slot_row = d->rows > 0 && pr.size > 0 ? pr.rows.get() : nullptr;  // nullptr: every slot empty
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
        lc.max_code += (plan->gcols[g].range - 1) * plan->gcols[g].stride;
      }
      fks[j] = fk.d;
      fkcols[j] = fk.view();
      probes[j] = &pr;
      elide[j] = ca.n_filters == 0 && ca.n_groups == 0 && link_covered(ctx, s, fk, *d, pk, pr);
      if (!elide[j]) note(fk);
    }
    // A link with no filter and no group column whose every fact key has a dim
    // row changes nothing in multiway_star_join (no fact row drops, nothing is
    // read from the dim): it is not scanned.  Removes its FK column read and its
    // per-row probe (SSB Q3.x joins part this way).
    {
      std::vector<laq_plan::LinkCode> kl;
      std::vector<const int32_t*> kf;
      std::vector<scan::Col> kc;
      std::vector<const Probe*> kp;
      for (int j = 0; j < q->n_joins; ++j)
        if (!elide[j]) {
          kl.push_back(std::move(plan->links[j]));
          kf.push_back(fks[j]);
          kc.push_back(fkcols[j]);
          kp.push_back(probes[j]);
        }
      plan->links = std::move(kl);
      fks = std::move(kf);
      fkcols = std::move(kc);
      probes = std::move(kp);
    }
    plan->nl = static_cast<int>(plan->links.size());
    plan->vec = aligned;
    plan->mode = G == 1 ? 0 : (G <= kSmemBinsPipe ? 1 : (G <= kSmemBinsLdg ? 1 : 2));
    plan->bytes_per_row = 4 * (plan->nl + plan->nf + a.n_fgroups + (a.measure ? 1 : 0));
    plan->packed_only = packed_only;
    plan->measure_min = mmin;
    lay_out_scan(ctx, plan.get(), fks, fkcols, probes, mmin, mmax, padded);
    if (packed_only && plan->variant != 2 && plan->variant != 4)
      fail(LAQ_ERR_UNSUPPORTED, "byte-packed fact columns need the stream scan (no fact InSet filter, G <= 4096)");
    {  // bit-packed columns (transfer format): only the direct kernel, and all-or-none
      int nbit = 0, ncol = 0;
      auto tally = [&](const scan::Col& c) { ++ncol; nbit += c.w == 0 ? 1 : 0; };
      if (a.measure) tally(a.mc);
      for (int j = 0; j < plan->nl; ++j) tally(a.fkc[j]);
      for (int f = 0; f < plan->nf; ++f) tally(a.ffc[f]);
      if (nbit > 0 && (nbit != ncol || plan->variant != 4 || a.n_fgroups > 0))
        fail(LAQ_ERR_UNSUPPORTED, "bit-packed fact columns need the direct scan with every scanned column bit-packed");
      if (nbit > 0) plan->variant = 6;
    }
    if (plan->variant == 6) {
      int64_t b = 0;  // bytes per row, rounded up per column
      if (a.measure) b += (a.mc.bits + 7) / 8;
      for (int j = 0; j < plan->nl; ++j) b += (a.fkc[j].bits + 7) / 8;
      for (int f = 0; f < plan->nf; ++f) b += (a.ffc[f].bits + 7) / 8;
      plan->bytes_per_row = b;
    }
    if (plan->variant == 2 || plan->variant == 4) {  // the stream kernels read the packed views
      bool any_packed = a.measure && a.mc.w != 4;
      for (int j = 0; j < plan->nl; ++j) any_packed = any_packed || a.fkc[j].w != 4;
      for (int f = 0; f < plan->nf; ++f) any_packed = any_packed || a.ffc[f].w != 4;
      if (any_packed) plan->variant += 1;
      int64_t b = 4 * a.n_fgroups + (a.measure ? a.mc.w : 0);
      for (int j = 0; j < plan->nl; ++j) b += a.fkc[j].w;
      for (int f = 0; f < plan->nf; ++f) b += a.ffc[f].w;
      plan->bytes_per_row = b;
    }
    if (plan->variant == 0 && plan->mode == 1 && G > kSmemBinsLdg) plan->mode = 2;
    *h_n_groups = G;
    *out = plan.release();
  });
}

int32_t laq_plan_scanned_links(const laq_plan* p) { return p ? p->nl : 0; }

int laq_plan_build_codes(laq_ctx* ctx, laq_plan* p) {
  return guard(ctx, [&] { build_codes(ctx, p); });
}

int laq_plans_build_codes(laq_ctx* ctx, int32_t n_plans, laq_plan* const* plans) {
  return guard(ctx, [&] {
    if (n_plans < 0) fail(LAQ_ERR_SHAPE, "negative plan count");
    if (build_codes_fused(ctx, plans, n_plans)) return;
    for (int i = 0; i < n_plans; ++i) build_codes(ctx, plans[i]);
  });
}

int laq_plan_scan(laq_ctx* ctx, laq_plan* p, int64_t* d_acc, int32_t accumulate) {
  return guard(ctx, [&] {
    if (!accumulate) LAQ_CUDA(cudaMemsetAsync(d_acc, 0, 2 * p->G * sizeof(int64_t), ctx->stream));
    if (p->fact_rows == 0) return;
    ScanArgs a = p->scan;
    a.acc = reinterpret_cast<unsigned long long*>(d_acc);
    launch_scan(ctx, a, p->nl, p->nf, p->mode, p->variant, p->vec, p->grid, p->smem);
  });
}

// Shared scan of a batch of plans (ssb_shared.cu).  Every plan must be a
// direct-kernel plan over the same int32 fact columns in the same roles (foreign
// keys, fact filters, measure); each plan's links and filters are re-ordered to
// the first plan's column order (the probe order changes, the result does not).
// Returns false when the batch does not qualify (the caller scans one by one).
static bool scan_shared(laq_ctx* ctx, int n, laq_plan* const* ps, int64_t* const* accs) {
  using namespace scan;
  if (n < 2 || n > kMaxShared || std::getenv("LAQ_NO_SHARED_SCAN")) return false;
  const laq_plan* p0 = ps[0];
  if (p0->variant != 4 || p0->fact_rows == 0) return false;
  // launch_shared instantiates 1..4 links and 0..2 fact filters; other shapes
  // take the one-plan-at-a-time path (same results).
  if (p0->nl < 1 || p0->nl > 4 || p0->nf > 2) return false;
  SharedScan M{};
  int optin = 0;
  LAQ_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  const int64_t budget = static_cast<int64_t>(optin) - 2048;
  int64_t off = 0;
  int64_t flush = INT64_MAX;
  int prefetch = 0;
  for (int q = 0; q < n; ++q) {
    const laq_plan* p = ps[q];
    const ScanArgs& a = p->scan;
    if (p->variant != 4 || p->nl != p0->nl || p->nf != p0->nf || p->mode != p0->mode || p->fact_rows != p0->fact_rows)
      return false;
    if (p->mode == 1 && !a.narrow_bins) return false;
    if ((a.measure == nullptr) != (p0->scan.measure == nullptr)) return false;
    if (a.measure && a.mc.p != p0->scan.mc.p) return false;
    ScanArgs b = a;
    // links: align to plan 0's fk columns
    bool used[kMaxLinks] = {};
    for (int j = 0; j < p0->nl; ++j) {
      int k = -1;
      for (int t = 0; t < p->nl && k < 0; ++t)
        if (!used[t] && a.fkc[t].p == p0->scan.fkc[j].p) k = t;
      if (k < 0) return false;
      used[k] = true;
      b.fk[j] = a.fk[k];
      b.fkc[j] = a.fkc[k];
      b.link[j] = a.link[k];
    }
    bool fused[kMaxFactFilters] = {};
    for (int f = 0; f < p0->nf; ++f) {
      int k = -1;
      for (int t = 0; t < p->nf && k < 0; ++t)
        if (!fused[t] && a.ffc[t].p == p0->scan.ffc[f].p) k = t;
      if (k < 0) return false;
      fused[k] = true;
      b.ff[f] = a.ff[k];
      b.ffc[f] = a.ffc[k];
    }
    // this query's staged tables, rebased after the previous queries'
    const int64_t base = off;
    for (int j = 0; j < p0->nl; ++j)
      if (b.link[j].fmt != kFmtGlobal) b.link[j].smem_byte += static_cast<int>(base);
    off += (a.smem_tab_elems + 15) & ~15;
    b.acc = reinterpret_cast<unsigned long long*>(accs[q]);
    M.q[q] = b;
    flush = std::min<int64_t>(flush, std::max<int64_t>(1, a.flush_every));
    prefetch = std::max(prefetch, a.prefetch);
  }
  for (int q = 0; q < n; ++q) {
    M.bins_off[q] = off;
    if (p0->mode == 1) off += 8 * ps[q]->G;
  }
  if (off > budget) return false;
  M.flush_every = flush;
  M.prefetch = prefetch;
  launch_shared(ctx, M, n, p0->nl, p0->nf, p0->mode, static_cast<size_t>(off));
  return true;
}

int laq_plans_scan_shared(laq_ctx* ctx, int32_t n_plans, laq_plan* const* plans, int64_t* const* d_accs,
                          int32_t accumulate, int32_t* h_shared) {
  return guard(ctx, [&] {
    if (n_plans < 0) fail(LAQ_ERR_SHAPE, "negative plan count");
    if (!accumulate)
      for (int q = 0; q < n_plans; ++q)
        LAQ_CUDA(cudaMemsetAsync(d_accs[q], 0, 2 * plans[q]->G * sizeof(int64_t), ctx->stream));
    const bool shared = scan_shared(ctx, n_plans, plans, d_accs);
    if (!shared)
      for (int q = 0; q < n_plans; ++q) {
        laq_plan* p = plans[q];
        if (p->fact_rows == 0) continue;
        ScanArgs a = p->scan;
        a.acc = reinterpret_cast<unsigned long long*>(d_accs[q]);
        launch_scan(ctx, a, p->nl, p->nf, p->mode, p->variant, p->vec, p->grid, p->smem);
      }
    if (h_shared) *h_shared = shared ? 1 : 0;
  });
}

int laq_plan_scan_range(laq_ctx* ctx, laq_plan* p, int64_t row0, int64_t rows, int64_t* d_acc, int32_t accumulate) {
  return guard(ctx, [&] {
    if (row0 < 0 || rows < 0 || row0 + rows > p->fact_rows) fail(LAQ_ERR_INDEX, "scan range outside the fact table");
    if (row0 % 4) fail(LAQ_ERR_SHAPE, "scan range must start at a multiple of 4 rows");
    if (!accumulate) LAQ_CUDA(cudaMemsetAsync(d_acc, 0, 2 * p->G * sizeof(int64_t), ctx->stream));
    if (rows == 0) return;
    ScanArgs a = p->scan;
    a.n = rows;
    auto shift = [&](scan::Col& c) {
      if (!c.p) return;
      if (c.w == 0) {  // bit-packed: whole 32-row groups of `bits` words
        if (row0 % 32) fail(LAQ_ERR_SHAPE, "scan range over bit-packed columns must start at a multiple of 32 rows");
        c.p = static_cast<const uint32_t*>(c.p) + (row0 / 32) * c.bits;
      } else {
        c.p = static_cast<const uint8_t*>(c.p) + row0 * c.w;
      }
    };
    for (int j = 0; j < p->nl; ++j) {
      if (a.fk[j]) a.fk[j] += row0;
      shift(a.fkc[j]);
    }
    for (int f = 0; f < p->nf; ++f) {
      if (a.ff[f].col) a.ff[f].col += row0;
      shift(a.ffc[f]);
    }
    for (int g = 0; g < a.n_fgroups; ++g) a.fg[g].col += row0;
    if (a.measure) {  // int32 column (other variants) or the stream kernel's "has a measure" flag
      a.measure += row0;
      shift(a.mc);
    }
    a.acc = reinterpret_cast<unsigned long long*>(d_acc);
    launch_scan(ctx, a, p->nl, p->nf, p->mode, p->variant, p->vec, p->grid, p->smem);
  });
}

int laq_plan_execute(laq_ctx* ctx, laq_plan* p, int64_t* d_acc, int32_t accumulate) {
  const int rc = laq_plan_build_codes(ctx, p);
  return rc ? rc : laq_plan_scan(ctx, p, d_acc, accumulate);
}

int64_t laq_plan_bytes_per_row(const laq_plan* p) { return p->bytes_per_row; }

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
    allreduce_i64(ctx, acc.get(), 2 * G);  // row-sharded: whole-table groups on every rank
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
    // prepare already built the code tables (pass fractions): scan only.
    const int rc2 = laq_plan_scan(ctx, p, ctx->d_flags + 32, 0);
    if (rc2) fail(rc2, ctx->err);
    int64_t rows = p->fact_rows;
    if (sharded(ctx)) {  // whole-table survivors / whole-table rows
      ctx->h_pinned[1] = p->fact_rows;
      LAQ_CUDA(cudaMemcpyAsync(ctx->d_flags + 33, ctx->h_pinned + 1, sizeof(int64_t), cudaMemcpyHostToDevice,
                               ctx->stream));
      allreduce_i64(ctx, ctx->d_flags + 32, 2);
      LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned + 1, ctx->d_flags + 33, sizeof(int64_t), cudaMemcpyDeviceToHost,
                               ctx->stream));
    }
    LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, ctx->d_flags + 32, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    if (sharded(ctx)) rows = ctx->h_pinned[1];
    *out = rows == 0 ? 0.0 : static_cast<double>(ctx->h_pinned[0]) / static_cast<double>(rows);
  });
  laq_plan_destroy(p);
  return rc;
}

}  // extern "C"

// ---- batched scan (ssb_batch.cuh): a batch of plans, one pass, one probe per link ----

struct laq_batch {
  laq_ctx* ctx = nullptr;
  std::vector<laq_plan*> plans;
  bool fused = false;
  std::string why;  // why the batch is scanned plan by plan (empty when fused)
  int nl = 0, nf = 0, mode = 0;
  scan::BatchScan B{};
  scan::DictArgs D{};
  DevMem<unsigned long long> hkeys;  // every link's hash table, one allocation
  DevMem<int32_t> hid;
  size_t hkey_count = 0;
  std::vector<DevMem<uint8_t>> ids;
  std::vector<DevMem<uint32_t>> bm;
  std::vector<DevMem<unsigned long long>> dec;
  DevMem<int> counts;  // [kBatchMaxLinks] tuple ids per link, [kBatchMaxLinks] overflow
  size_t smem = 0;
  int grid = 1;
  int64_t bytes_per_row = 0;
  std::vector<int> n_dec;
};

namespace laq {
namespace {

int ceil_log2(int64_t v) {
  int b = 0;
  while ((int64_t{1} << b) < v) ++b;
  return b;
}

// (Re)allocate the dictionary of every link: hash tables sized for `cap`
// tuples per link, id tables of width idw[j], decode tables of cap[j] entries.
void batch_alloc_dict(laq_batch* b, const std::vector<int64_t>& cap, const std::vector<int>& idw,
                      const std::vector<char>& want_bm) {
  scan::DictArgs& D = b->D;
  size_t total = 0;
  std::vector<int> hb(b->nl);
  for (int j = 0; j < b->nl; ++j) {
    hb[j] = std::max(6, ceil_log2(2 * cap[j]));
    total += size_t{1} << hb[j];
  }
  b->hkeys = DevMem<unsigned long long>(total);
  b->hid = DevMem<int32_t>(total);
  b->hkey_count = total;
  b->ids.clear();
  b->bm.clear();
  b->dec.clear();
  size_t off = 0;
  for (int j = 0; j < b->nl; ++j) {
    scan::DictLink& L = D.l[j];
    L.hkeys = b->hkeys.get() + off;
    L.hid = b->hid.get() + off;
    L.hbits = hb[j];
    off += size_t{1} << hb[j];
    L.idw = idw[j];
    b->ids.emplace_back(static_cast<size_t>((((L.slots + 1) * idw[j]) + 15) & ~int64_t{15}));
    L.ids = b->ids.back().get();
    b->dec.emplace_back(static_cast<size_t>((cap[j] + 1) & ~int64_t{1}));  // 16-byte multiple
    L.dec = b->dec.back().get();
    L.dec_cap = static_cast<int>(cap[j]);
    if (want_bm[j]) {
      b->bm.emplace_back(static_cast<size_t>((((L.slots + 32) / 32) + 3) & ~int64_t{3}));
      L.bm = b->bm.back().get();
    } else {
      b->bm.emplace_back();
      L.bm = nullptr;
    }
  }
}

void batch_build(laq_ctx* ctx, laq_batch* b, bool dict) {
  const int n = static_cast<int>(b->plans.size());
  if (!build_codes_fused(ctx, b->plans.data(), n))
    for (auto* p : b->plans) build_codes(ctx, p);
  if (!dict) return;
  LAQ_CUDA(cudaMemsetAsync(b->hkeys.get(), 0xFF, b->hkey_count * sizeof(unsigned long long), ctx->stream));
  LAQ_CUDA(cudaMemsetAsync(b->counts.get(), 0, 2 * scan::kBatchMaxLinks * sizeof(int), ctx->stream));
  scan::launch_dict_build(ctx, b->D);
}

// Decide whether a batch runs fused and lay it out; b->why says why not.
void batch_prepare(laq_ctx* ctx, laq_batch* b) {
  using namespace scan;
  const int nq = static_cast<int>(b->plans.size());
  auto reject = [&](const std::string& why) {
    b->fused = false;
    b->why = why;
  };
  if (std::getenv("LAQ_NO_BATCH_SCAN")) return reject("LAQ_NO_BATCH_SCAN");
  if (nq < 2 || nq > kBatchMaxQ) return reject("the fused pass takes batches of 2..4 plans");
  const laq_plan* p0 = b->plans[0];
  if (p0->fact_rows == 0) return reject("empty fact table");
  int mode = 0;
  for (const laq_plan* p : b->plans) {
    const ScanArgs& a = p->scan;
    if (p->variant != 4) return reject("a plan is not on the direct int32 scan");
    if (p->fact_rows != p0->fact_rows) return reject("plans over different fact tables");
    if (p->mode > 1 || (p->mode == 1 && !a.narrow_bins)) return reject("wide group bins");
    if (p->G > kLaneFail) return reject("more than 4096 groups");
    if ((a.measure == nullptr) != (p0->scan.measure == nullptr) || (a.measure && a.mc.p != p0->scan.mc.p))
      return reject("different measures");
    if (a.measure && a.mc.w != 4) return reject("packed measure");
    mode = std::max(mode, p->mode);
  }
  // Bins with a positive measure: sums only (a group is present iff its sum
  // is non-zero), half the shared atomics of (count, sum) bins: SF=100 Q3
  // group 1.77 -> 1.45 ms; Q4 group (L2-gathered part ids) 3.13 -> 3.10 ms,
  // same box, with the current kernel (an earlier one measured it slower there).
  bool positive_measure = false;
  if (mode == 1 && p0->scan.measure) {
    bool positive = true;
    for (const laq_plan* p : b->plans) positive = positive && p->measure_min > 0;
    positive_measure = positive && !std::getenv("LAQ_BATCH_COUNT_BINS");
  }
  // Union of links (keyed by the fact FK column) and of fact filter columns.
  struct U {
    const void* col;
    Col c;
    uint32_t base, size;
    int64_t slots;
    const int32_t* code[kBatchMaxQ];
  };
  std::vector<U> links;
  std::vector<std::pair<const void*, Col>> fcols;
  int32_t flo[kBatchMaxFilters][kBatchMaxQ], fhi[kBatchMaxFilters][kBatchMaxQ];
  uint32_t reject_mask = 0;
  for (int f = 0; f < kBatchMaxFilters; ++f)
    for (int q = 0; q < kBatchMaxQ; ++q) flo[f][q] = INT32_MIN, fhi[f][q] = INT32_MAX;
  for (int q = 0; q < nq; ++q) {
    const laq_plan* p = b->plans[q];
    const ScanArgs& a = p->scan;
    for (int t = 0; t < p->nl; ++t) {
      const LinkProbe& lp = a.link[t];
      if (lp.kind != PROBE_DIRECT || a.fkc[t].w != 4) return reject("non-direct link or packed key column");
      int u = -1;
      for (size_t k = 0; k < links.size(); ++k)
        if (links[k].col == a.fkc[t].p) u = static_cast<int>(k);
      if (u < 0) {
        if (links.size() == static_cast<size_t>(kBatchMaxLinks)) return reject("more than 6 distinct links");
        U x{a.fkc[t].p, a.fkc[t], static_cast<uint32_t>(lp.base), static_cast<uint32_t>(lp.size),
            std::max<int64_t>(lp.size, 1), {}};
        links.push_back(x);
        u = static_cast<int>(links.size()) - 1;
      }
      U& x = links[u];
      if (x.base != static_cast<uint32_t>(lp.base) || x.size != static_cast<uint32_t>(lp.size))
        return reject("one FK column probed into different dimensions");
      if (x.code[q]) return reject("a plan joins one FK column twice");
      x.code[q] = lp.code;
    }
    for (int f = 0; f < p->nf; ++f) {
      const FactFilter& ff = a.ff[f];
      if (ff.inset || a.ffc[f].w != 4) return reject("InSet or packed fact filter");
      int u = -1;
      for (size_t k = 0; k < fcols.size(); ++k)
        if (fcols[k].first == a.ffc[f].p) u = static_cast<int>(k);
      if (u < 0) {
        if (fcols.size() == 2) return reject("more than 2 fact filter columns");
        fcols.emplace_back(a.ffc[f].p, a.ffc[f]);
        u = static_cast<int>(fcols.size()) - 1;
      }
      if (ff.lo > ff.hi) reject_mask |= 1u << q;  // an empty interval: the query matches no row
      flo[u][q] = std::max(flo[u][q], ff.lo);
      fhi[u][q] = std::min(fhi[u][q], ff.hi);
      if (flo[u][q] > fhi[u][q]) reject_mask |= 1u << q;
    }
  }
  if (links.empty()) return reject("no links");
  b->nl = static_cast<int>(links.size());
  b->nf = static_cast<int>(fcols.size());
  b->mode = mode;

  // Dictionaries, first pass: room for every slot's tuple (uint16 ids).
  DictArgs& D = b->D;
  D = DictArgs{};
  D.nl = b->nl;
  D.nq = nq;
  b->counts = DevMem<int>(2 * kBatchMaxLinks);
  D.n_dec = b->counts.get();
  D.overflow = b->counts.get() + kBatchMaxLinks;
  std::vector<int64_t> cap(b->nl);
  for (int j = 0; j < b->nl; ++j) {
    DictLink& L = D.l[j];
    L.slots = links[j].slots;
    L.size = links[j].size;
    unsigned long long miss = 0;
    for (int q = 0; q < nq; ++q) {
      L.code[q] = links[j].code[q];
      if (L.code[q]) miss |= static_cast<unsigned long long>(kLaneFail) << (16 * q);
    }
    L.miss = miss;
    D.start[j + 1] = D.start[j] + ((L.slots + 1 + 31) & ~int64_t{31});  // covers the miss slot `size`
    cap[j] = std::min<int64_t>(L.slots + 1, 65536);
  }
  batch_alloc_dict(b, cap, std::vector<int>(b->nl, 2), std::vector<char>(b->nl, 0));
  batch_build(ctx, b, true);
  int h[2 * kBatchMaxLinks];
  LAQ_CUDA(cudaMemcpyAsync(h, b->counts.get(), sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  for (int j = 0; j < b->nl; ++j)
    if (h[kBatchMaxLinks]) return reject("more than 65535 distinct code tuples on a link");
  b->n_dec.assign(h, h + b->nl);

  // Pass fraction of each link (slots some joining query keeps), host side, once.
  std::vector<double> frac(b->nl, 1.0);
  for (int j = 0; j < b->nl; ++j) {
    const DictLink& L = D.l[j];
    std::vector<uint16_t> ids(static_cast<size_t>(L.slots));
    std::vector<unsigned long long> dec(static_cast<size_t>(b->n_dec[j]));
    LAQ_CUDA(cudaMemcpy(ids.data(), L.ids, ids.size() * 2, cudaMemcpyDeviceToHost));
    LAQ_CUDA(cudaMemcpy(dec.data(), L.dec, dec.size() * 8, cudaMemcpyDeviceToHost));
    std::vector<char> keep(dec.size(), 0);
    for (size_t t = 0; t < dec.size(); ++t)
      for (int q = 0; q < nq; ++q)
        if (L.code[q] && ((dec[t] >> (16 * q)) & 0xFFFF) < kLaneFail) keep[t] = 1;
    int64_t k = 0;
    for (uint16_t v : ids) k += keep[v];
    frac[j] = static_cast<double>(k) / static_cast<double>(std::max<int64_t>(L.slots, 1));
  }

  // Shared-memory layout: bins, decode tables, then id tables smallest first,
  // then any-pass bitmaps for the links left in global memory.
  int optin = 0;
  LAQ_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  int64_t room = static_cast<int64_t>(optin) - 2048;
  int64_t bins = 0;
  const int64_t bin_words = mode == 1 ? 2 : 1;  // u32 words per group (room reserved for (count, sum) bins)
  if (mode != 0)
    for (const laq_plan* p : b->plans) bins += (4 * bin_words * p->G + 15) & ~int64_t{15};
  // Narrow decode (4-byte entries, 3 x 10-bit lanes) when every lane fits:
  // contributions < fail32 (a power of two >= every G) and at most
  // (links + fact filters + 1) fails: G - 1 + (nl + nf + 1) * fail32 < 1024.
  int64_t max_g = 1;
  for (const laq_plan* p : b->plans) max_g = std::max<int64_t>(max_g, p->G);
  int64_t f32 = 1;
  while (f32 < max_g) f32 <<= 1;
  const bool dec32 = nq <= 3 && b->nl <= 3 && !std::getenv("LAQ_BATCH_PIPE") && !std::getenv("LAQ_BATCH_DEC64") &&
                     (max_g - 1) + (b->nl + b->nf + 1) * f32 <= 1023;
  const int64_t dec_entry = dec32 ? 4 : 8;
  std::vector<int64_t> decb(b->nl), idb(b->nl), bmb(b->nl);
  std::vector<int> idw(b->nl);
  for (int j = 0; j < b->nl; ++j) {
    decb[j] = (dec_entry * int64_t{b->n_dec[j]} + 15) & ~int64_t{15};
    idw[j] = b->n_dec[j] <= 256 ? 1 : 2;
    idb[j] = ((D.l[j].slots + 1) * idw[j] + 15) & ~int64_t{15};
    bmb[j] = (((D.l[j].slots + 32) / 32) * 4 + 15) & ~int64_t{15};
    room -= decb[j];
  }
  room -= bins;
  if (room < 0) return reject("decode tables and bins exceed shared memory");
  std::vector<int> by(b->nl);
  std::iota(by.begin(), by.end(), 0);
  std::stable_sort(by.begin(), by.end(), [&](int x, int y) { return idb[x] < idb[y]; });
  std::vector<char> staged(b->nl, 0), use_bm(b->nl, 0);
  if (std::getenv("LAQ_BATCH_BITMAP_FIRST") && b->nl > 0) {
    // A/B knob: the largest link keeps only its any-pass bitmap in shared
    // memory (its ids gathered through L2) before the id tables are placed.
    const int big = by.back();
    if (bmb[big] <= room && frac[big] < 0.75) use_bm[big] = 1, room -= bmb[big];
  }
  for (int j : by)
    if (!std::getenv("LAQ_NOSMEMTAB") && !use_bm[j] && idb[j] <= room) staged[j] = 1, room -= idb[j];
  for (int j : by)
    if (!staged[j] && !use_bm[j] && bmb[j] <= room && frac[j] < 0.75) use_bm[j] = 1, room -= bmb[j];
  // Probe order: shared-memory links first, then L2 gathers; most selective first.
  std::vector<int> order(b->nl);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
    if (staged[x] != staged[y]) return staged[x] > staged[y];
    return frac[x] < frac[y];
  });
  // Joint pair: the first two probe-order links, both staged, share one decode
  // table of n0 x n1 entries (one decode load per row instead of two) when it
  // is small and fits; sum-bin (positive measure) batches, the instantiated form.
  std::vector<int64_t> dec_n(b->n_dec.begin(), b->n_dec.end());  // entries staged per link
  bool joint = false;
  // Only when every link is staged: with an L2-gathered link the pass is bound by
  // the gathers and the smaller decode replication the joint table leaves costs
  // more than the saved load (SF=100 Q4 group 3.14 vs 3.10 ms; Q3 group 1.38 vs
  // 1.45 ms with it, profiles/round2/batch_ab_joint_pair.json).
  // The pair is the two staged links with the fewest joint entries, moved to
  // the front of the probe order (staged links commute; gathered links keep
  // their place after them).  With a gathered link the pair must be small
  // enough to keep the decode replication (LAQ_BATCH_JOINT_GATHER_MAX entries,
  // default 64: SF=100 Q4's commitdate x orderdate = 45).
  bool all_staged = true;
  for (int j = 0; j < b->nl; ++j) all_staged = all_staged && staged[j];
  int64_t pair_max = all_staged ? 1024 : 64;
  if (!all_staged)
    if (const char* e = std::getenv("LAQ_BATCH_JOINT_GATHER_MAX")) pair_max = std::atoll(e);
  const bool want_joint = positive_measure && b->nl >= 2 && !std::getenv("LAQ_BATCH_PIPE") &&
                          !std::getenv("LAQ_BATCH_NOJOINT");
  int q0 = -1, q1 = -1;
  for (int x = 0; want_joint && x < b->nl; ++x)
    for (int y = x + 1; y < b->nl; ++y)
      if (staged[order[x]] && staged[order[y]] &&
          (q0 < 0 || int64_t{b->n_dec[order[x]]} * b->n_dec[order[y]] <
                         int64_t{b->n_dec[order[q0]]} * b->n_dec[order[q1]]))
        q0 = x, q1 = y;
  if (q0 >= 0 && int64_t{b->n_dec[order[q0]]} * b->n_dec[order[q1]] <= pair_max) {
    const int a0 = order[q0], a1 = order[q1];
    std::vector<int> rest;
    for (int x = 0; x < b->nl; ++x)
      if (x != q0 && x != q1) rest.push_back(order[x]);
    order.assign({a0, a1});
    order.insert(order.end(), rest.begin(), rest.end());
  }
  if (want_joint && staged[order[0]] && staged[order[1]] &&
      int64_t{b->n_dec[order[0]]} * b->n_dec[order[1]] <= pair_max) {
    const int o0 = order[0], o1 = order[1];
    const int64_t nj = int64_t{b->n_dec[o0]} * b->n_dec[o1];
    const int64_t jb = (dec_entry * nj + 15) & ~int64_t{15};
    if (nj <= 1024 && jb - decb[o0] - decb[o1] <= room) {
      room -= jb - decb[o0] - decb[o1];
      decb[o0] = 0;
      decb[o1] = jb;
      dec_n[o0] = 0;
      dec_n[o1] = nj;
      joint = true;
    }
  }
  // Decode tables replicated `rep` times (entry-interleaved) with what room is
  // left: lane l reads copy l % rep, so a warp's 32 random decodes conflict at
  // most 32/rep-way on a bank instead of colliding on the few entries' banks.
  int rep = 1;
  {
    int64_t dec_total = 0;
    for (int j = 0; j < b->nl; ++j) dec_total += decb[j];
    while (rep < 16 && dec_total * (2 * rep - rep) <= room) {
      room -= dec_total * rep;
      rep *= 2;
    }
    if (const char* e = std::getenv("LAQ_BATCH_DEC_REP")) rep = std::max(1, std::min(rep, std::atoi(e)));
  }

  if (positive_measure) mode = 2;
  b->mode = mode;
  const int64_t final_bin_words = mode == 1 ? 2 : 1;
  // Final dictionaries: exact capacities and id widths.
  for (int j = 0; j < b->nl; ++j) cap[j] = b->n_dec[j];
  batch_alloc_dict(b, cap, idw, use_bm);

  BatchScan& B = b->B;
  B = BatchScan{};
  B.n = p0->fact_rows;
  B.nq = nq;
  int64_t off = 0;
  bool gathers = false;
  for (int t = 0; t < b->nl; ++t) {  // kernel link t = union link order[t]
    const int j = order[t];
    const DictLink& L = D.l[j];
    BatchLink& K = B.link[t];
    K.base = links[j].base;
    K.size = links[j].size;
    K.miss = static_cast<uint32_t>(b->n_dec[j] - 1);
    K.ids = L.ids;
    K.dec = L.dec;
    K.bm = L.bm;
    K.fmt = staged[j] ? (idw[j] == 1 ? kIdSmemU8 : kIdSmemU16) : (idw[j] == 1 ? kIdGlobU8 : kIdGlobU16);
    K.dec_byte = static_cast<int>(off);
    K.n_dec = static_cast<int>(dec_n[j]);
    off += decb[j] * rep;
    B.fkc[t] = links[j].c;
    gathers = gathers || !staged[j];
  }
  for (int t = 0; t < b->nl; ++t) {
    const int j = order[t];
    BatchLink& K = B.link[t];
    K.id_byte = 0;
    K.id_bytes = 0;
    if (staged[j]) {
      K.id_byte = static_cast<int>(off);
      K.id_bytes = static_cast<int>(idb[j]);
      off += idb[j];
    }
    K.bm_byte = -1;
    if (use_bm[j]) {
      K.bm_byte = static_cast<int>(off);
      K.bm_bytes = static_cast<int>(bmb[j]);
      off += bmb[j];
    }
  }
  for (int f = 0; f < b->nf; ++f) {
    B.ffc[f] = fcols[f].second;
    for (int q = 0; q < kBatchMaxQ; ++q) B.ff_lo[f][q] = flo[f][q], B.ff_hi[f][q] = fhi[f][q];
  }
  B.has_measure = p0->scan.measure ? 1 : 0;
  B.mc = p0->scan.mc;
  int64_t flush = INT64_MAX;
  for (int q = 0; q < nq; ++q) {
    const laq_plan* p = b->plans[q];
    B.G[q] = p->G;
    if (mode != 0) {
      B.bins_byte[q] = static_cast<int>(off);
      off += (4 * final_bin_words * p->G + 15) & ~int64_t{15};
    }
    flush = std::min<int64_t>(flush, std::max<int64_t>(1, p->scan.flush_every));
  }
  B.init_lo = B.init_hi = B.fail_lo = B.fail_hi = 0;
  B.dec32 = dec32 ? 1 : 0;
  B.joint01 = joint ? 1 : 0;
  B.n_tup1 = joint ? static_cast<uint32_t>(b->n_dec[order[1]]) : 1u;
  B.fail32 = static_cast<uint32_t>(f32);
  for (int q = 0; q < nq; ++q) {
    if (dec32) {
      B.fail_lo += static_cast<uint32_t>(f32) << (10 * q);
      if (reject_mask & (1u << q)) B.init_lo += static_cast<uint32_t>(f32) << (10 * q);
      continue;
    }
    const uint32_t f = kLaneFail << (16 * (q & 1));
    (q < 2 ? B.fail_lo : B.fail_hi) += f;
    if (reject_mask & (1u << q)) (q < 2 ? B.init_lo : B.init_hi) += f;
  }
  // Software pipelining of the last link's L2 gather (scan_batch_pipe_kernel,
  // 2 rows per thread) when that link is gathered: opt-in (LAQ_BATCH_PIPE=1).
  // It removes the gather stalls (long-scoreboard 33 % -> 5 %) but doubles the
  // per-row instruction count: SF=100 Q4 group 3.22 -> 3.48 ms, issue-bound.
  B.pipe = !staged[order[b->nl - 1]] && mode != 0 && std::getenv("LAQ_BATCH_PIPE") ? 1 : 0;

  B.dec_shift = dec32 ? 2 : 3;  // log2(entry bytes * rep)
  while ((1 << (B.dec_shift - (dec32 ? 2 : 3))) < rep) ++B.dec_shift;
  B.flush_every = flush;
  B.prefetch = gathers ? 2 : 0;
  if (const char* pf = std::getenv("LAQ_PREFETCH")) B.prefetch = std::atoi(pf);
  b->smem = static_cast<size_t>(off);
  b->grid = ctx->sm_count;
  b->bytes_per_row = 4 * (b->nl + b->nf + B.has_measure);
  b->fused = true;
  b->why.clear();
  if (std::getenv("LAQ_BATCH_VERBOSE")) {
    std::fprintf(stderr, "[laq batch] nq=%d nl=%d nf=%d mode=%d dec32=%d rep=%d smem=%lld joint01=%d\n", nq, b->nl,
                 b->nf, mode, dec32 ? 1 : 0, rep, static_cast<long long>(off), joint ? 1 : 0);
    for (int t = 0; t < b->nl; ++t) {
      const int j = order[t];
      std::fprintf(stderr, "[laq batch]   link %d: slots=%lld tuples=%d frac=%.3f fmt=%d id_bytes=%d bm_bytes=%d\n", t,
                   static_cast<long long>(D.l[j].slots), b->n_dec[j], frac[j], B.link[t].fmt, B.link[t].id_bytes,
                   B.link[t].bm_byte >= 0 ? B.link[t].bm_bytes : 0);
    }
  }
  batch_build(ctx, b, true);  // leave the batch ready to scan
}

}  // namespace
}  // namespace laq

extern "C" {

int laq_batch_prepare(laq_ctx* ctx, int32_t n_plans, laq_plan* const* plans, laq_batch** out, int32_t* h_fused) {
  return guard(ctx, [&] {
    if (n_plans < 1) fail(LAQ_ERR_SHAPE, "empty plan batch");
    auto b = std::make_unique<laq_batch>();
    b->ctx = ctx;
    b->plans.assign(plans, plans + n_plans);
    batch_prepare(ctx, b.get());
    if (!b->fused) {
      b->hkeys = DevMem<unsigned long long>();
      b->ids.clear();
      b->dec.clear();
      b->bm.clear();
    }
    if (h_fused) *h_fused = b->fused ? 1 : 0;
    *out = b.release();
  });
}

int laq_batch_build(laq_ctx* ctx, laq_batch* b) {
  return guard(ctx, [&] { batch_build(ctx, b, b->fused); });
}

int laq_batch_scan(laq_ctx* ctx, laq_batch* b, int64_t* const* d_accs, int32_t accumulate) {
  return guard(ctx, [&] {
    const int nq = static_cast<int>(b->plans.size());
    if (!accumulate)
      for (int q = 0; q < nq; ++q)
        LAQ_CUDA(cudaMemsetAsync(d_accs[q], 0, 2 * b->plans[q]->G * sizeof(int64_t), ctx->stream));
    if (b->fused) {
      scan::BatchScan B = b->B;
      for (int q = 0; q < nq; ++q) B.acc[q] = reinterpret_cast<unsigned long long*>(d_accs[q]);
      scan::launch_batch(ctx, B, b->nl, b->nf, b->mode, b->smem, b->grid);
      return;
    }
    for (int q = 0; q < nq; ++q) {
      laq_plan* p = b->plans[q];
      if (p->fact_rows == 0) continue;
      ScanArgs a = p->scan;
      a.acc = reinterpret_cast<unsigned long long*>(d_accs[q]);
      launch_scan(ctx, a, p->nl, p->nf, p->mode, p->variant, p->vec, p->grid, p->smem);
    }
  });
}

int laq_batch_info(const laq_batch* b, int32_t* fused, int64_t* bytes_per_row, int32_t* n_links, char* why,
                   size_t why_cap) {
  if (!b) return LAQ_ERR_GENERIC;
  if (fused) *fused = b->fused ? 1 : 0;
  if (bytes_per_row) {
    int64_t s = 0;
    for (const laq_plan* p : b->plans) s += p->bytes_per_row;
    *bytes_per_row = b->fused ? b->bytes_per_row : s;
  }
  if (n_links) *n_links = b->nl;
  if (why && why_cap) {
    std::strncpy(why, b->why.c_str(), why_cap - 1);
    why[why_cap - 1] = 0;
  }
  return LAQ_OK;
}

int laq_batch_destroy(laq_batch* b) {
  delete b;
  return LAQ_OK;
}

}  // extern "C"
