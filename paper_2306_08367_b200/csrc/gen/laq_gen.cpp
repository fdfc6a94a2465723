// Host-side synthetic data generator: a bit-exact restatement of the
// reference's generator (proj/src/benchgen.cpp:13-199, proj/include/laq/rng.hpp)
// so the GPU engine and the CPU reference consume identical arrays.
//
// Not on the hot path (generation stays on the host); it is
// native C++ because SF=100 means 4.8e9 draws.  The reference's Rng::bounded
// (rng.hpp:25-31) does a 64-bit modulo per draw; we replace the hardware
// divide by an exact multiply-high (Granlund–Montgomery) that returns the same
// remainder for every 64-bit input (checked in tests/test_gen.py), which is
// what makes SF=100 generation take seconds instead of minutes.
//
// Columns can be emitted as int64 (the reference's IntColumn) or narrowed to
// int32 (the device layout); every generated value fits int32.

#include <algorithm>
#include <bit>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

// ---- rng.hpp:9-51 ---------------------------------------------------------
inline std::uint64_t fnv1a(const char* s, std::size_t n, std::uint64_t h = 0xcbf29ce484222325ull) {
  for (std::size_t i = 0; i < n; ++i) {
    h ^= static_cast<unsigned char>(s[i]);
    h *= 0x100000001b3ull;
  }
  return h;
}
inline std::uint64_t derive_seed(std::uint64_t seed, const std::string& tag) {
  return seed ^ fnv1a(tag.data(), tag.size());
}

// Exact x % n for 64-bit x via a precomputed reciprocal.
struct FastMod {
  std::uint64_t n = 1, magic = 0;
  int shift = 0;
  bool pow2 = false, add = false;
  explicit FastMod(std::uint64_t d = 1) : n(d) {
    if (d == 0) return;
    if ((d & (d - 1)) == 0) {
      pow2 = true;
      shift = std::countr_zero(d);
      return;
    }
    const int l = 63 - std::countl_zero(d);
    const unsigned __int128 num = static_cast<unsigned __int128>(1) << (64 + l);
    std::uint64_t m = static_cast<std::uint64_t>(num / d);
    const std::uint64_t rem = static_cast<std::uint64_t>(num % d);
    const std::uint64_t e = d - rem;
    if (e < (std::uint64_t{1} << l)) {
      shift = l;
    } else {
      m += m;
      const std::uint64_t twice = rem + rem;
      if (twice >= d || twice < rem) m += 1;
      shift = l;
      add = true;
    }
    magic = m + 1;
  }
  inline std::uint64_t div(std::uint64_t x) const {
    if (pow2) return x >> shift;
    const std::uint64_t q = static_cast<std::uint64_t>((static_cast<unsigned __int128>(magic) * x) >> 64);
    if (add) {
      const std::uint64_t t = ((x - q) >> 1) + q;
      return t >> (shift);
    }
    return q >> shift;
  }
  inline std::uint64_t mod(std::uint64_t x) const { return x - div(x) * n; }
};

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : e_(seed) {}
  std::uint64_t next() { return e_(); }
  // rng.hpp:25-31 with a fixed modulus.
  struct Bounded {
    FastMod fm;
    std::uint64_t limit;
    explicit Bounded(std::uint64_t n)
        : fm(n), limit(n ? UINT64_MAX - (UINT64_MAX % n) : 0) {}
  };
  std::uint64_t bounded(const Bounded& b) {
    if (b.fm.n == 0) return 0;
    std::uint64_t x = e_();
    while (x >= b.limit) x = e_();
    return b.fm.mod(x);
  }
  double unit() { return static_cast<double>(e_() >> 11) * 0x1.0p-53; }  // rng.hpp:39

 private:
  std::mt19937_64 e_;
};

constexpr std::int64_t kCategoryRange = 25, kBrandRange = 40, kSizeRange = 1000, kRegionRange = 5,
                       kNationRange = 25, kCityRange = 250, kRankRange = 1000, kYearLo = 1992,
                       kYearHi = 1999, kDayRange = 365, kDateRows = 7 * 365;  // benchgen.cpp:17-26

struct Col {
  std::string name;
  int kind;  // 0 key, 1 int, 2 float (storage.hpp:14)
  std::vector<std::int64_t> i64;
  std::vector<std::int32_t> i32;
  std::vector<double> f64;
};

struct Tab {
  std::string name;
  std::int64_t rows = 0;
  std::vector<Col> cols;
};

struct Star {
  std::vector<Tab> tables;  // [lineorder, part, supplier, date, (customer)]
  bool narrow = false;
};

// Row window of the fact table a generator call keeps: all n values are drawn
// (the engine stream must advance exactly as in the reference, one column
// after the other), only rows [lo, hi) are stored.  The default keeps all.
struct Window {
  std::int64_t lo = 0, hi = INT64_MAX;
};

// Emit an integer column through a per-value generator.
template <class F>
void fill_int(Col& c, std::int64_t n, bool narrow, F&& f, Window w = {}) {
  const std::int64_t lo = std::min(w.lo, n), hi = std::max(lo, std::min(w.hi, n));
  for (std::int64_t i = 0; i < lo; ++i) (void)f();
  if (narrow) {
    c.i32.resize(static_cast<std::size_t>(hi - lo));
    for (std::int64_t i = lo; i < hi; ++i) c.i32[i - lo] = static_cast<std::int32_t>(f());
  } else {
    c.i64.resize(static_cast<std::size_t>(hi - lo));
    for (std::int64_t i = lo; i < hi; ++i) c.i64[i - lo] = f();
  }
  for (std::int64_t i = hi; i < n; ++i) (void)f();
}

void uniform_col(Col& c, Rng& rng, std::int64_t n, std::int64_t lo, std::int64_t hi, bool narrow, Window w = {}) {
  const Rng::Bounded b(static_cast<std::uint64_t>(hi - lo));
  fill_int(c, n, narrow, [&] { return lo + static_cast<std::int64_t>(rng.bounded(b)); }, w);
}

void iota_col(Col& c, std::int64_t n, bool narrow) {
  std::int64_t v = 0;
  fill_int(c, n, narrow, [&] { return v++; });
}

// benchgen.cpp:46-55
void fk_col(Col& c, Rng& rng, std::int64_t n, std::int64_t dim_rows, double dangling, bool narrow, Window w = {}) {
  const Rng::Bounded b(static_cast<std::uint64_t>(dim_rows));
  fill_int(c, n, narrow, [&] {
    const bool miss = dangling > 0.0 && rng.unit() < dangling;
    return static_cast<std::int64_t>(rng.bounded(b)) + (miss ? dim_rows : 0);
  }, w);
}

std::vector<std::int64_t> split_features(std::int64_t k, std::size_t parts) {  // benchgen.cpp:57-61
  std::vector<std::int64_t> out(parts, k / static_cast<std::int64_t>(parts));
  for (std::int64_t i = 0; i < k % static_cast<std::int64_t>(parts); ++i) ++out[i];
  return out;
}

// benchgen.cpp:63-101
Tab make_dim(const std::string& name, char prefix, std::int64_t rows, std::int64_t features,
             std::uint64_t seed, bool narrow) {
  Rng rng(derive_seed(seed, name));
  Tab t;
  t.name = name;
  t.rows = rows;
  const std::string p(1, prefix);
  auto add = [&](const std::string& n, int kind) -> Col& {
    t.cols.push_back(Col{n, kind, {}, {}, {}});
    return t.cols.back();
  };
  iota_col(add(p + "_key", 0), rows, narrow);
  if (name == "date") {
    uniform_col(add("d_year", 1), rng, rows, kYearLo, kYearHi, narrow);
    uniform_col(add("d_month", 1), rng, rows, 1, 13, narrow);
    uniform_col(add("d_dayofyear", 1), rng, rows, 0, kDayRange, narrow);
  } else if (name == "part") {
    uniform_col(add("p_category", 1), rng, rows, 0, kCategoryRange, narrow);
    uniform_col(add("p_brand", 1), rng, rows, 0, kBrandRange, narrow);
    uniform_col(add("p_size", 1), rng, rows, 0, kSizeRange, narrow);
  } else {
    uniform_col(add(p + "_region", 1), rng, rows, 0, kRegionRange, narrow);
    uniform_col(add(p + "_nation", 1), rng, rows, 0, kNationRange, narrow);
    uniform_col(add(p + "_city", 1), rng, rows, 0, kCityRange, narrow);
    uniform_col(add(p + "_rank", 1), rng, rows, 0, kRankRange, narrow);
  }
  for (std::int64_t f = 0; f < features; ++f) {
    Col& c = add(p + "_f" + std::to_string(f), 2);
    c.f64.resize(static_cast<std::size_t>(rows));
    for (auto& v : c.f64) v = rng.unit();
  }
  return t;
}

struct Card {
  std::int64_t lineorder = 0, part = 0, supplier = 0, customer = 0, date = 0;
};

Card cardinalities(int setting, std::int64_t sf) {  // benchgen.cpp:165-188
  const auto log_scale = static_cast<std::int64_t>(std::bit_width(static_cast<std::uint64_t>(sf)));
  Card c;
  c.date = kDateRows;
  c.supplier = sf * 2000;
  if (setting == 0) {
    c.lineorder = sf * 600000;
    c.part = 20000 * log_scale;
  } else if (setting == 1) {
    c.lineorder = sf * 3000;
    c.part = 2000 * log_scale;
  } else {
    c.lineorder = sf * 6000000;
    c.part = 200000 * log_scale;
    c.customer = sf * 30000;
  }
  return c;
}

}  // namespace

extern "C" {

typedef struct laqgen_star laqgen_star;

const char* laqgen_last_error() { return g_err.c_str(); }

// setting: 0 = S1, 1 = S2, 2 = Ssb.  Status codes follow include/laq_b200.h
// (12 = GenError, 13 = CapacityError).  max_bytes <= 0 means the reference's
// default cap of 4 GiB (benchgen.hpp:280).
// fact_tag != NULL draws lineorder from derive_seed(seed, "lineorder/<tag>")
// instead of "lineorder": an independent fact shard over the SAME dimension
// tables (weak-scaling runs give every GPU its own SF-sized shard).
// row_lo / row_hi: keep only lineorder rows [row_lo, row_hi) of the canonical
// table (a contiguous row shard for multi-GPU runs: every rank draws the same
// stream and stores its own rows, so the shards concatenate to exactly the
// reference's table).  row_hi < 0 keeps everything.
int laqgen_star_create_shard(int setting, std::int64_t sf, std::uint64_t seed, std::int64_t feature_width,
                             double dangling, std::int64_t max_bytes, int narrow32, const char* fact_tag,
                             std::int64_t row_lo, std::int64_t row_hi, laqgen_star** out) {
  try {
    if (sf < 1) { g_err = "scale factor must be >= 1"; return 12; }
    if (feature_width < 0) { g_err = "feature width must be >= 0"; return 12; }
    const bool with_customer = setting == 2;
    const Card card = cardinalities(setting, sf);
    if (max_bytes <= 0) max_bytes = std::int64_t{4} << 30;
    // benchgen.cpp:113-123 capacity guard (8 bytes per stored value)
    const auto feats = split_features(feature_width, 3);
    const std::int64_t fact_cols = with_customer ? 8 : 7;
    std::int64_t cells = card.lineorder * fact_cols;
    cells += card.part * (4 + feats[0]);
    cells += card.supplier * (5 + feats[1]);
    cells += card.date * (4 + feats[2]);
    if (with_customer) cells += card.customer * 5;
    if (cells * 8 > max_bytes) {
      g_err = "dataset needs " + std::to_string(cells * 8) + " bytes, cap is " + std::to_string(max_bytes);
      return 13;
    }
    Window w;
    if (row_hi >= 0) {
      if (row_lo < 0 || row_lo > row_hi || row_hi > card.lineorder) {
        g_err = "fact row window out of range";
        return 12;
      }
      w.lo = row_lo;
      w.hi = row_hi;
    }
    const bool narrow = narrow32 != 0;
    auto s = std::make_unique<Star>();
    s->narrow = narrow;
    s->tables.resize(with_customer ? 5 : 4);
    // Dimensions draw from their own engines: build them concurrently with the fact.
    std::thread dims([&] {
      s->tables[1] = make_dim("part", 'p', card.part, feats[0], seed, narrow);
      s->tables[2] = make_dim("supplier", 's', card.supplier, feats[1], seed, narrow);
      s->tables[3] = make_dim("date", 'd', card.date, feats[2], seed, narrow);
      if (with_customer) s->tables[4] = make_dim("customer", 'c', card.customer, 0, seed, narrow);
    });
    {  // benchgen.cpp:132-152: one engine, columns in order
      Rng rng(derive_seed(seed, fact_tag ? std::string("lineorder/") + fact_tag : std::string("lineorder")));
      Tab& t = s->tables[0];
      t.name = "lineorder";
      t.rows = std::min(w.hi, card.lineorder) - std::min(w.lo, card.lineorder);
      t.cols.reserve(8);
      auto add = [&](const char* n, int kind) -> Col& {
        t.cols.push_back(Col{n, kind, {}, {}, {}});
        return t.cols.back();
      };
      const std::int64_t n = card.lineorder;
      fk_col(add("lo_part", 0), rng, n, card.part, dangling, narrow, w);
      fk_col(add("lo_supplier", 0), rng, n, card.supplier, dangling, narrow, w);
      fk_col(add("lo_orderdate", 0), rng, n, card.date, dangling, narrow, w);
      fk_col(add("lo_commitdate", 0), rng, n, card.date, dangling, narrow, w);
      if (with_customer) fk_col(add("lo_customer", 0), rng, n, card.customer, dangling, narrow, w);
      uniform_col(add("lo_quantity", 1), rng, n, 1, 51, narrow, w);
      uniform_col(add("lo_discount", 1), rng, n, 0, 11, narrow, w);
      uniform_col(add("lo_revenue", 1), rng, n, 100, 10000, narrow, w);
    }
    dims.join();
    *out = reinterpret_cast<laqgen_star*>(s.release());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int laqgen_star_create_tagged(int setting, std::int64_t sf, std::uint64_t seed, std::int64_t feature_width,
                              double dangling, std::int64_t max_bytes, int narrow32, const char* fact_tag,
                              laqgen_star** out) {
  return laqgen_star_create_shard(setting, sf, seed, feature_width, dangling, max_bytes, narrow32, fact_tag, 0, -1,
                                  out);
}

int laqgen_star_create(int setting, std::int64_t sf, std::uint64_t seed, std::int64_t feature_width,
                       double dangling, std::int64_t max_bytes, int narrow32, laqgen_star** out) {
  return laqgen_star_create_tagged(setting, sf, seed, feature_width, dangling, max_bytes, narrow32, nullptr, out);
}

void laqgen_star_destroy(laqgen_star* s) { delete reinterpret_cast<Star*>(s); }
int laqgen_n_tables(const laqgen_star* s) {
  return static_cast<int>(reinterpret_cast<const Star*>(s)->tables.size());
}
const char* laqgen_table_name(const laqgen_star* s, int t) {
  return reinterpret_cast<const Star*>(s)->tables[t].name.c_str();
}
std::int64_t laqgen_table_rows(const laqgen_star* s, int t) {
  return reinterpret_cast<const Star*>(s)->tables[t].rows;
}
int laqgen_table_ncols(const laqgen_star* s, int t) {
  return static_cast<int>(reinterpret_cast<const Star*>(s)->tables[t].cols.size());
}
const char* laqgen_col_name(const laqgen_star* s, int t, int c) {
  return reinterpret_cast<const Star*>(s)->tables[t].cols[c].name.c_str();
}
int laqgen_col_kind(const laqgen_star* s, int t, int c) {
  return reinterpret_cast<const Star*>(s)->tables[t].cols[c].kind;
}
// Element size in bytes of the column's storage (4 = int32, 8 = int64/double).
int laqgen_col_width(const laqgen_star* s, int t, int c) {
  const Star* st = reinterpret_cast<const Star*>(s);
  return st->tables[t].cols[c].kind == 2 ? 8 : (st->narrow ? 4 : 8);
}
const void* laqgen_col_data(const laqgen_star* s, int t, int c) {
  const Star* st = reinterpret_cast<const Star*>(s);
  const Col& col = st->tables[t].cols[c];
  if (col.kind == 2) return col.f64.data();
  return st->narrow ? static_cast<const void*>(col.i32.data()) : static_cast<const void*>(col.i64.data());
}

// gen_linear (benchgen.cpp:512-518): k x l row-major, uniform [-1, 1).
int laqgen_gen_linear(std::int64_t k, std::int64_t l, std::uint64_t seed, double* out) {
  if (k < 1 || l < 1) { g_err = "gen_linear: need positive shape"; return 12; }
  Rng rng(derive_seed(seed, "linear"));
  for (std::int64_t i = 0; i < k * l; ++i) out[i] = rng.unit() * 2.0 - 1.0;
  return 0;
}

// Raw draws for the configs that have no reference generator entry point
// (cfg1: fk = Rng(derive_seed(seed, tag)).range(lo, hi) x n).
int laqgen_range(std::uint64_t seed, const char* tag, std::int64_t n, std::int64_t lo, std::int64_t hi,
                 std::int64_t* out64, std::int32_t* out32) {
  Rng rng(tag ? derive_seed(seed, tag) : seed);
  const Rng::Bounded b(static_cast<std::uint64_t>(hi - lo));
  for (std::int64_t i = 0; i < n; ++i) {
    const std::int64_t v = lo + static_cast<std::int64_t>(rng.bounded(b));
    if (out64) out64[i] = v;
    if (out32) out32[i] = static_cast<std::int32_t>(v);
  }
  return 0;
}

// Column-by-column unit() draws, as make_dim does for feature columns
// (benchgen.cpp:96-99); out is row-major rows x cols.
int laqgen_unit_matrix(std::uint64_t seed, const char* tag, std::int64_t rows, std::int64_t cols, double* out) {
  Rng rng(tag ? derive_seed(seed, tag) : seed);
  for (std::int64_t c = 0; c < cols; ++c)
    for (std::int64_t r = 0; r < rows; ++r) out[r * cols + c] = rng.unit();
  return 0;
}

// Test hook: exact fast modulo vs hardware modulo.
std::uint64_t laqgen_fastmod(std::uint64_t x, std::uint64_t n) { return FastMod(n).mod(x); }

}  // extern "C"
