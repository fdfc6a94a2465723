// TEST INFRASTRUCTURE ONLY — C-ABI into the UNMODIFIED reference library.
//
// This file is ours; everything it calls is the reference's own code compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/.  It lets
// the Python tests (ctypes) and bench.py's CPU legs (cpu_baseline and
// --impl reference) run the reference implementation on the same host arrays
// the GPU engine consumes.  Never linked into the product library.
//
// Every wrapper catches laq::Error and returns the status code that
// include/laq_b200.h assigns to that subclass, so the two implementations can
// be compared error-for-error.

#include <algorithm>
#include <chrono>
#include <cstring>
#include <map>
#include <numeric>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "../include/laq_b200.h"
#include "laq/benchgen.hpp"
#include "laq/cli.hpp"
#include "laq/fusion.hpp"
#include "laq/laqops.hpp"
#include "laq/oracle.hpp"
#include "laq/report.hpp"
#include "laq/rng.hpp"

using namespace laq;

namespace {

thread_local std::string g_err;

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return LAQ_OK;
  } catch (const CapacityError& e) { g_err = e.what(); return LAQ_ERR_CAPACITY;
  } catch (const GenError& e) { g_err = e.what(); return LAQ_ERR_GEN;
  } catch (const ModelError& e) { g_err = e.what(); return LAQ_ERR_MODEL;
  } catch (const TreeError& e) { g_err = e.what(); return LAQ_ERR_TREE;
  } catch (const DuplicateKeyError& e) { g_err = e.what(); return LAQ_ERR_DUPLICATE_KEY;
  } catch (const DomainError& e) { g_err = e.what(); return LAQ_ERR_DOMAIN;
  } catch (const MappingError& e) { g_err = e.what(); return LAQ_ERR_MAPPING;
  } catch (const TypeError& e) { g_err = e.what(); return LAQ_ERR_TYPE;
  } catch (const NameError& e) { g_err = e.what(); return LAQ_ERR_NAME;
  } catch (const FormatError& e) { g_err = e.what(); return LAQ_ERR_FORMAT;
  } catch (const ShapeError& e) { g_err = e.what(); return LAQ_ERR_SHAPE;
  } catch (const IndexError& e) { g_err = e.what(); return LAQ_ERR_INDEX;
  } catch (const Error& e) { g_err = e.what(); return LAQ_ERR_GENERIC;
  } catch (const std::exception& e) { g_err = e.what(); return LAQ_ERR_GENERIC; }
}

// A StarSchema plus a flat view of its tables: index 0 is the fact table.
struct RefStar {
  StarSchema star;
  std::vector<std::string> names;
  std::vector<const Table*> tables;
  // Row-sharded copies (for the multi-threaded CPU baseline).
  std::vector<StarSchema> shards;

  void index() {
    names.clear();
    tables.clear();
    names.push_back("lineorder");
    tables.push_back(&star.fact());
    for (const auto& [name, t] : star.dims()) {
      names.push_back(name);
      tables.push_back(&t);
    }
  }
};

Predicate to_pred(const laq_filter_desc& f) {
  if (f.is_float) {
    const double lo = static_cast<double>(f.lo), hi = static_cast<double>(f.hi);
    switch (f.kind) {
      case LAQ_PRED_LT: return Predicate::lt(lo);
      case LAQ_PRED_LE: return Predicate::le(lo);
      case LAQ_PRED_EQ: return Predicate::eq(lo);
      case LAQ_PRED_GE: return Predicate::ge(lo);
      case LAQ_PRED_GT: return Predicate::gt(lo);
      case LAQ_PRED_BETWEEN: return Predicate::between(lo, hi);
      default: {
        std::vector<double> v;
        for (int64_t i = 0; i < f.set_len; ++i) v.push_back(static_cast<double>(f.set[i]));
        return Predicate::in_set(std::move(v));
      }
    }
  }
  switch (f.kind) {
    case LAQ_PRED_LT: return Predicate::lt(std::int64_t{f.lo});
    case LAQ_PRED_LE: return Predicate::le(std::int64_t{f.lo});
    case LAQ_PRED_EQ: return Predicate::eq(std::int64_t{f.lo});
    case LAQ_PRED_GE: return Predicate::ge(std::int64_t{f.lo});
    case LAQ_PRED_GT: return Predicate::gt(std::int64_t{f.lo});
    case LAQ_PRED_BETWEEN: return Predicate::between(std::int64_t{f.lo}, std::int64_t{f.hi});
    default: return Predicate::in_set(std::vector<std::int64_t>(f.set, f.set + f.set_len));
  }
}

bench::QuerySpec to_spec(const laq_query_desc& d) {
  bench::QuerySpec q;
  q.id = "capi";
  for (int i = 0; i < d.n_joins; ++i)
    q.joins.push_back({d.joins[i].fact_fk, d.joins[i].dim_name, d.joins[i].dim_pk});
  for (int i = 0; i < d.n_filters; ++i)
    q.filters.push_back({d.filters[i].target, d.filters[i].column, to_pred(d.filters[i])});
  q.measure = d.measure ? d.measure : "lo_revenue";
  for (int i = 0; i < d.n_group; ++i) q.group_by.push_back({d.group_by[i].target, d.group_by[i].column});
  q.order_by = d.order_by != 0;
  return q;
}

int copy_out(const DenseMat& m, double* out, int64_t cap, int64_t* rows, int64_t* cols) {
  *rows = m.rows();
  *cols = m.cols();
  if (m.rows() * m.cols() > cap) {
    g_err = "output capacity";
    return LAQ_ERR_CAPACITY;
  }
  std::copy(m.data().begin(), m.data().end(), out);
  return LAQ_OK;
}

Table key_table(const int64_t* keys, int64_t n, const char* name) {
  return Table(Schema{{name, ColKind::Key}}, {IntColumn(keys, keys + n)});
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- generator (benchgen.cpp:103-199) -----------------------------------
void* ref_gen_star(int setting, int64_t sf, uint64_t seed, int64_t feature_width, double dangling,
                   int64_t max_bytes) {
  RefStar* h = nullptr;
  const int rc = guard([&] {
    bench::GenConfig cfg;
    cfg.sf = sf;
    cfg.setting = setting == 0 ? bench::Setting::S1 : setting == 1 ? bench::Setting::S2 : bench::Setting::Ssb;
    cfg.seed = seed;
    cfg.feature_width = feature_width;
    cfg.dangling_fraction = dangling;
    if (max_bytes > 0) cfg.max_bytes = max_bytes;
    h = new RefStar{bench::gen_star(cfg), {}, {}, {}};
    h->index();
  });
  return rc == LAQ_OK ? h : nullptr;
}

// ---- dataset files (cli.cpp:430-481 write_dataset, storage.cpp:112-150 load_csv) ----
int ref_write_dataset(int setting, int64_t sf, uint64_t seed, int64_t feature_width, double dangling,
                      const char* dir) {
  return guard([&] {
    bench::GenConfig cfg;
    cfg.sf = sf;
    cfg.setting = setting == 0 ? bench::Setting::S1 : setting == 1 ? bench::Setting::S2 : bench::Setting::Ssb;
    cfg.seed = seed;
    cfg.feature_width = feature_width;
    cfg.dangling_fraction = dangling;
    cli::write_dataset(bench::gen_star(cfg), cfg, std::nullopt, dir);
  });
}

// load_csv into caller buffers (int64 for key/int, double for float; kinds per
// storage.hpp:14 order Key=0, Int=1, Float=2).  *rows = rows read; LAQ_ERR_CAPACITY
// if more than cap.
int ref_load_csv(const char* path, int ncols, const int32_t* kinds, int64_t cap, void* const* out, int64_t* rows) {
  return guard([&] {
    Schema sc;
    for (int c = 0; c < ncols; ++c)
      sc.columns.emplace_back("c" + std::to_string(c), kinds[c] == 0 ? ColKind::Key : kinds[c] == 1 ? ColKind::Int
                                                                                                    : ColKind::Float);
    const Table t = load_csv(path, sc);
    *rows = t.row_count();
    if (t.row_count() > cap) throw CapacityError("ref_load_csv: capacity");
    for (int c = 0; c < ncols; ++c) {
      if (kinds[c] == 2)
        std::memcpy(out[c], t.floats(c).data(), t.row_count() * sizeof(double));
      else
        std::memcpy(out[c], t.ints(c).data(), t.row_count() * sizeof(int64_t));
    }
  });
}

void ref_star_free(void* h) { delete static_cast<RefStar*>(h); }
int ref_star_n_tables(void* h) { return static_cast<int>(static_cast<RefStar*>(h)->tables.size()); }
const char* ref_star_table_name(void* h, int t) { return static_cast<RefStar*>(h)->names[t].c_str(); }
int64_t ref_star_table_rows(void* h, int t) { return static_cast<RefStar*>(h)->tables[t]->row_count(); }
int ref_star_table_ncols(void* h, int t) { return static_cast<int>(static_cast<RefStar*>(h)->tables[t]->col_count()); }
const char* ref_star_col_name(void* h, int t, int c) {
  return static_cast<RefStar*>(h)->tables[t]->schema().name(c).c_str();
}
int ref_star_col_kind(void* h, int t, int c) {
  return static_cast<int>(static_cast<RefStar*>(h)->tables[t]->schema().kind(c));
}
const void* ref_star_col_data(void* h, int t, int c) {
  const Table* tb = static_cast<RefStar*>(h)->tables[t];
  if (tb->schema().kind(c) == ColKind::Float) return tb->floats(c).data();
  return tb->ints(c).data();
}

// Build a star from raw host columns (tests).  Tables: [fact, dims...];
// kinds per storage.hpp:14; links name fact fk / dim / pk.
void* ref_star_from_columns(int n_tables, const char* const* names, const int64_t* rows,
                            const int* ncols, const char* const* const* col_names,
                            const int* const* kinds, const void* const* const* cols, int n_links,
                            const laq_link_desc* links) {
  RefStar* h = nullptr;
  const int rc = guard([&] {
    std::vector<Table> tables;
    for (int t = 0; t < n_tables; ++t) {
      Schema s;
      std::vector<Column> cs;
      for (int c = 0; c < ncols[t]; ++c) {
        const ColKind k = static_cast<ColKind>(kinds[t][c]);
        s.columns.emplace_back(col_names[t][c], k);
        if (k == ColKind::Float) {
          const double* p = static_cast<const double*>(cols[t][c]);
          cs.emplace_back(FloatColumn(p, p + rows[t]));
        } else {
          const int64_t* p = static_cast<const int64_t*>(cols[t][c]);
          cs.emplace_back(IntColumn(p, p + rows[t]));
        }
      }
      tables.emplace_back(std::move(s), std::move(cs));
    }
    std::vector<std::pair<std::string, Table>> dims;
    for (int t = 1; t < n_tables; ++t) dims.emplace_back(names[t], std::move(tables[t]));
    std::vector<StarLink> ls;
    for (int i = 0; i < n_links; ++i) ls.push_back({links[i].fact_fk, links[i].dim_name, links[i].dim_pk});
    h = new RefStar{StarSchema(std::move(tables[0]), std::move(dims), std::move(ls)), {}, {}, {}};
    h->index();
  });
  return rc == LAQ_OK ? h : nullptr;
}

// ---- query driver (cli.cpp:73-232) --------------------------------------
// engine 0 = run_query_laq, 1 = run_query_oracle.
int ref_run_query(void* h, const laq_query_desc* d, int engine, double* out, int64_t cap,
                  int64_t* rows, int64_t* cols, double* seconds) {
  int inner = LAQ_OK;
  const int rc = guard([&] {
    RefStar* s = static_cast<RefStar*>(h);
    const bench::QuerySpec q = to_spec(*d);
    const double t0 = now_s();
    const DenseMat m = engine == 0 ? cli::run_query_laq(s->star, q) : cli::run_query_oracle(s->star, q);
    if (seconds) *seconds = now_s() - t0;
    inner = copy_out(m, out, cap, rows, cols);
  });
  return rc != LAQ_OK ? rc : inner;
}

int ref_measure_selectivity(void* h, const laq_query_desc* d, double* out) {
  return guard([&] { *out = bench::measure_selectivity(static_cast<RefStar*>(h)->star, to_spec(*d)); });
}

// gen_queries (benchgen.cpp:413-457): tuned dial constants of the group's
// three queries (the dial filter is the last filter, `column < C`).
int ref_gen_queries(void* h, int group, const double* targets, int n_targets, int64_t* dials,
                    double* realized) {
  return guard([&] {
    const std::vector<double> t(targets, targets + n_targets);
    const auto qs = bench::gen_queries(static_cast<RefStar*>(h)->star,
                                       static_cast<bench::QueryGroup>(group), t);
    for (std::size_t i = 0; i < qs.size(); ++i) {
      realized[i] = qs[i].realized_selectivity;
      // The dial is the appended Lt predicate; recover its constant by probing.
      const Predicate& p = qs[i].filters.back().pred;
      int64_t lo = 0, hi = 1 << 20;
      while (lo < hi) {  // smallest v with !(v < C)  ==> v == C
        const int64_t mid = lo + (hi - lo) / 2;
        if (p.matches(mid)) lo = mid + 1; else hi = mid;
      }
      dials[i] = lo;
    }
  });
}

// Multi-threaded CPU baseline: the fact table split into contiguous row
// shards, run_query_laq per shard on its own thread, group sums merged.  Only
// valid for SUM queries (sums are additive), which is every workload query.
int ref_star_make_shards(void* h, int n_shards) {
  return guard([&] {
    RefStar* s = static_cast<RefStar*>(h);
    s->shards.clear();
    const Table& fact = s->star.fact();
    const int64_t n = fact.row_count();
    for (int k = 0; k < n_shards; ++k) {
      const int64_t b = n * k / n_shards, e = n * (k + 1) / n_shards;
      std::vector<Column> cs;
      for (index_t c = 0; c < fact.col_count(); ++c) {
        if (fact.schema().kind(c) == ColKind::Float) {
          const auto& src = fact.floats(c);
          cs.emplace_back(FloatColumn(src.begin() + b, src.begin() + e));
        } else {
          const auto& src = fact.ints(c);
          cs.emplace_back(IntColumn(src.begin() + b, src.begin() + e));
        }
      }
      std::vector<std::pair<std::string, Table>> dims(s->star.dims().begin(), s->star.dims().end());
      s->shards.emplace_back(Table(fact.schema(), std::move(cs)), std::move(dims), s->star.links());
    }
  });
}

int ref_run_query_sharded(void* h, const laq_query_desc* d, int engine, double* out, int64_t cap,
                          int64_t* rows, int64_t* cols, double* seconds) {
  int inner = LAQ_OK;
  const int rc = guard([&] {
    RefStar* s = static_cast<RefStar*>(h);
    const bench::QuerySpec q = to_spec(*d);
    const std::size_t n = s->shards.size();
    std::vector<DenseMat> parts(n);
    std::vector<std::string> errs(n);
    const double t0 = now_s();
    std::vector<std::thread> th;
    for (std::size_t k = 0; k < n; ++k)
      th.emplace_back([&, k] {
        try {
          parts[k] = engine == 0 ? cli::run_query_laq(s->shards[k], q) : cli::run_query_oracle(s->shards[k], q);
        } catch (const std::exception& e) { errs[k] = e.what(); }
      });
    for (auto& t : th) t.join();
    for (auto& e : errs)
      if (!e.empty()) throw Error(e);
    // Merge: rows keyed by group tuple (all columns but the last).
    std::map<std::vector<double>, double> acc;
    const index_t w = parts.empty() ? 1 : parts[0].cols();
    for (const DenseMat& p : parts)
      for (index_t r = 0; r < p.rows(); ++r) {
        std::vector<double> key(p.row(r), p.row(r) + (w - 1));
        acc[key] += p(r, w - 1);
      }
    DenseMat m(static_cast<index_t>(acc.size()), w);
    index_t r = 0;
    for (const auto& [key, sum] : acc) {
      for (index_t c = 0; c + 1 < w; ++c) m(r, c) = key[c];
      m(r, w - 1) = sum;
      ++r;
    }
    if (seconds) *seconds = now_s() - t0;
    inner = copy_out(m, out, cap, rows, cols);
  });
  return rc != LAQ_OK ? rc : inner;
}

// ---- key encoding and joins (laqops.cpp:123-319) -------------------------
int ref_build_key_domain(const int64_t* r, int64_t nr, const int64_t* s, int64_t ns, int64_t* out,
                         int64_t* n) {
  return guard([&] {
    const auto d = ops::build_key_domain({r, static_cast<size_t>(nr)}, {s, static_cast<size_t>(ns)});
    std::copy(d.sorted_keys.begin(), d.sorted_keys.end(), out);
    *n = d.size();
  });
}

int ref_update_key_domain(const int64_t* dom, int64_t nd, const int64_t* nk, int64_t nn,
                          int64_t* out, int64_t* n) {
  return guard([&] {
    const auto base = ops::build_key_domain({dom, static_cast<size_t>(nd)}, {});
    const auto d = ops::update_key_domain(base, {nk, static_cast<size_t>(nn)});
    std::copy(d.sorted_keys.begin(), d.sorted_keys.end(), out);
    *n = d.size();
  });
}

// orientation 0 = RowsByDomain, 1 = DomainByRows.  vals may be NULL.
int ref_key_matrix(const int64_t* keys, int64_t n, const int64_t* dom, int64_t nd, int orientation,
                   const double* vals, int64_t* row_ptr, int64_t* col_idx, double* values,
                   int64_t* nnz, int64_t* rows) {
  return guard([&] {
    const auto d = ops::build_key_domain({dom, static_cast<size_t>(nd)}, {});
    std::span<const double> v;
    if (vals) v = {vals, static_cast<size_t>(n)};
    const SparseCsr m = ops::key_matrix({keys, static_cast<size_t>(n)}, d,
                                        orientation == 0 ? ops::KeyOrientation::RowsByDomain
                                                         : ops::KeyOrientation::DomainByRows,
                                        v);
    std::copy(m.row_ptr.begin(), m.row_ptr.end(), row_ptr);
    std::copy(m.col_idx.begin(), m.col_idx.end(), col_idx);
    std::copy(m.values.begin(), m.values.end(), values);
    *nnz = m.nnz();
    *rows = m.rows;
  });
}

int ref_mm_join(const int64_t* r, int64_t nr, const int64_t* s, int64_t ns, int64_t* out_r,
                int64_t* out_s, int64_t cap, int64_t* nnz) {
  int inner = LAQ_OK;
  const int rc = guard([&] {
    const ops::RowMatch m = ops::mm_join({r, static_cast<size_t>(nr)}, {s, static_cast<size_t>(ns)});
    *nnz = m.nnz();
    if (m.nnz() > cap) {
      inner = LAQ_ERR_CAPACITY;
      return;
    }
    std::copy(m.mat.row_idx.begin(), m.mat.row_idx.end(), out_r);
    std::copy(m.mat.col_idx.begin(), m.mat.col_idx.end(), out_s);
  });
  return rc != LAQ_OK ? rc : inner;
}

// multiway_star_join over raw key arrays: fact columns f0..f{J-1}, dims with pk "k".
int ref_star_join(int n_links, const int64_t* const* fks, int64_t n, const int64_t* const* pks,
                  const int64_t* pk_rows, int64_t* surv, int64_t* const* dim_rows, int64_t* nnz,
                  double* seconds) {
  return guard([&] {
    Schema fs;
    std::vector<Column> fc;
    std::vector<std::string> fnames;
    for (int j = 0; j < n_links; ++j) {
      fnames.push_back("f" + std::to_string(j));
      fs.columns.emplace_back(fnames.back(), ColKind::Key);
      fc.emplace_back(IntColumn(fks[j], fks[j] + n));
    }
    const Table fact(fs, std::move(fc));
    std::vector<Table> dims;
    dims.reserve(n_links);
    for (int j = 0; j < n_links; ++j) dims.push_back(key_table(pks[j], pk_rows[j], "k"));
    std::vector<ops::DimJoinSpec> specs;
    for (int j = 0; j < n_links; ++j) specs.push_back({&dims[j], fnames[j], "k"});
    std::vector<index_t> survivors;
    const double t0 = now_s();
    const auto got = ops::multiway_star_join(fact, specs, &survivors);
    if (seconds) *seconds = now_s() - t0;
    *nnz = static_cast<int64_t>(survivors.size());
    if (surv) std::copy(survivors.begin(), survivors.end(), surv);
    for (int j = 0; j < n_links; ++j)
      if (dim_rows && dim_rows[j]) std::copy(got[j].mat.col_idx.begin(), got[j].mat.col_idx.end(), dim_rows[j]);
  });
}

// oracle::star_join (oracle.cpp:63-109), many-to-many expansion order.
int ref_oracle_star_join(int n_links, const int64_t* const* fks, int64_t n, const int64_t* const* pks,
                         const int64_t* pk_rows, int64_t* fact_rows, int64_t* const* dim_rows,
                         int64_t cap, int64_t* nnz) {
  int inner = LAQ_OK;
  const int rc = guard([&] {
    Schema fs;
    std::vector<Column> fc;
    std::vector<std::string> fnames;
    for (int j = 0; j < n_links; ++j) {
      fnames.push_back("f" + std::to_string(j));
      fs.columns.emplace_back(fnames.back(), ColKind::Key);
      fc.emplace_back(IntColumn(fks[j], fks[j] + n));
    }
    const Table fact(fs, std::move(fc));
    std::vector<Table> dims;
    for (int j = 0; j < n_links; ++j) dims.push_back(key_table(pks[j], pk_rows[j], "k"));
    std::vector<oracle::DimRef> refs;
    for (int j = 0; j < n_links; ++j) refs.push_back({&dims[j], fnames[j], "k"});
    const oracle::StarMatch m = oracle::star_join(fact, refs);
    *nnz = m.row_count();
    if (m.row_count() > cap) { inner = LAQ_ERR_CAPACITY; return; }
    std::copy(m.fact_rows.begin(), m.fact_rows.end(), fact_rows);
    for (int j = 0; j < n_links; ++j) std::copy(m.dim_rows[j].begin(), m.dim_rows[j].end(), dim_rows[j]);
  });
  return rc != LAQ_OK ? rc : inner;
}

// ---- aggregation (laqops.cpp:376-455) ------------------------------------
int ref_groupby_sum_single(const int64_t* kr, const double* vr, int64_t nr, const int64_t* ks,
                           const int64_t* gs, int64_t ns, int64_t* out_g, double* out_s, int64_t* n) {
  return guard([&] {
    const auto res = ops::groupby_sum_single({kr, static_cast<size_t>(nr)}, {vr, static_cast<size_t>(nr)},
                                             {ks, static_cast<size_t>(ns)}, {gs, static_cast<size_t>(ns)});
    for (std::size_t g = 0; g < res.size(); ++g) {
      out_g[g] = res[g].group;
      out_s[g] = res[g].sum;
    }
    *n = static_cast<int64_t>(res.size());
  });
}

int ref_groupby_sum_multi(int n_cols, const int64_t* const* cols, const double* vals, int64_t n,
                          int64_t* out_keys, double* out_sums, int64_t cap, int64_t* n_groups) {
  return guard([&] {
    std::vector<IntColumn> gc;
    for (int c = 0; c < n_cols; ++c) gc.emplace_back(cols[c], cols[c] + n);
    const auto res = ops::groupby_sum_multi(gc, {vals, static_cast<size_t>(n)});
    *n_groups = static_cast<int64_t>(res.size());
    for (std::size_t g = 0; g < res.size(); ++g) {
      for (int c = 0; c < n_cols; ++c) out_keys[c * cap + static_cast<int64_t>(g)] = res[g].group[c];
      out_sums[g] = res[g].sum;
    }
  });
}

// ---- fusion (fusion.cpp:31-77) and the non-fused plan ---------------------
namespace {
struct StarMats {
  std::vector<DenseMat> dims;
  std::vector<ops::ColumnMap> maps;
  std::vector<SparseCsr> imaps;
};
StarMats make_mats(int n_dims, const double* const* dims, const int64_t* rows, const int64_t* cols,
                   const int64_t* const* placements, int64_t k, const int64_t* const* idx, int64_t m) {
  StarMats s;
  for (int j = 0; j < n_dims; ++j) {
    s.dims.emplace_back(rows[j], cols[j], std::vector<double>(dims[j], dims[j] + rows[j] * cols[j]));
    std::vector<std::pair<index_t, index_t>> mapping;
    for (int64_t c = 0; c < cols[j]; ++c) mapping.emplace_back(c, placements[j][c]);
    s.maps.push_back(ops::build_placement_map(cols[j], k, mapping));
    if (idx) {
      SparseCsr im;
      im.rows = m;
      im.cols = rows[j];
      im.row_ptr.resize(static_cast<size_t>(m) + 1);
      std::iota(im.row_ptr.begin(), im.row_ptr.end(), index_t{0});
      im.col_idx.assign(idx[j], idx[j] + m);
      im.values.assign(static_cast<size_t>(m), 1.0);
      s.imaps.push_back(std::move(im));
    }
  }
  return s;
}
}  // namespace

int ref_prefuse_linear(int n_dims, const double* const* dims, const int64_t* rows, const int64_t* cols,
                       const int64_t* const* placements, const double* L, int64_t k, int64_t l,
                       double* const* partials) {
  return guard([&] {
    StarMats s = make_mats(n_dims, dims, rows, cols, placements, k, nullptr, 0);
    ml::LinearOperator op{DenseMat(k, l, std::vector<double>(L, L + k * l))};
    const auto f = fusion::prefuse_linear(s.dims, s.maps, op);
    for (int j = 0; j < n_dims; ++j) std::copy(f.partials[j].data().begin(), f.partials[j].data().end(), partials[j]);
  });
}

int ref_apply_fused_linear(int n_parts, const int64_t* const* idx, int64_t m, const double* const* partials,
                           const int64_t* prow, int64_t l, double* out) {
  return guard([&] {
    fusion::FusedLinear f;
    f.out_width = l;
    std::vector<SparseCsr> imaps;
    for (int j = 0; j < n_parts; ++j) {
      f.partials.emplace_back(prow[j], l, std::vector<double>(partials[j], partials[j] + prow[j] * l));
      SparseCsr im;
      im.rows = m;
      im.cols = prow[j];
      im.row_ptr.resize(static_cast<size_t>(m) + 1);
      std::iota(im.row_ptr.begin(), im.row_ptr.end(), index_t{0});
      im.col_idx.assign(idx[j], idx[j] + m);
      im.values.assign(static_cast<size_t>(m), 1.0);
      imaps.push_back(std::move(im));
    }
    const DenseMat y = fusion::apply_fused_linear(imaps, f);
    std::copy(y.data().begin(), y.data().end(), out);
  });
}

// Non-fused plan: materialize (laqops.cpp:338-374) + predict_linear (mlops.cpp:248-250).
int ref_materialize_predict(int n_dims, const double* const* dims, const int64_t* rows,
                            const int64_t* cols, const int64_t* const* placements, int64_t k,
                            const int64_t* const* idx, int64_t m, const double* L, int64_t l,
                            double* out_T, double* out_Y) {
  return guard([&] {
    StarMats s = make_mats(n_dims, dims, rows, cols, placements, k, idx, m);
    const DenseMat t = ops::materialize(s.imaps, s.dims, s.maps);
    if (out_T) std::copy(t.data().begin(), t.data().end(), out_T);
    if (out_Y) {
      ml::LinearOperator op{DenseMat(k, l, std::vector<double>(L, L + k * l))};
      const DenseMat y = ml::predict_linear(t, op);
      std::copy(y.data().begin(), y.data().end(), out_Y);
    }
  });
}

int ref_dense_matmul(const double* a, int64_t m, int64_t k, const double* b, int64_t n, double* c) {
  return guard([&] {
    const DenseMat A(m, k, std::vector<double>(a, a + m * k));
    const DenseMat B(k, n, std::vector<double>(b, b + k * n));
    const DenseMat C = dense_matmul(A, B);
    std::copy(C.data().begin(), C.data().end(), c);
  });
}

// The cfg1 fused pipeline through the reference API:
// multiway_star_join -> csr_from_coo -> prefuse_linear -> apply_fused_linear.
// One dim per link, dim features B_j (r_j x k_j) placed contiguously.
// seconds[0..3] = join, csr, prefuse, apply.
// cfg1 inputs drawn with the REFERENCE's own Rng (rng.hpp) and
// gen_linear (benchgen.cpp:512-518), for bench.py's reference arm: fk =
// Rng(derive_seed(seed, "lineorder")).range(0, dim_rows) x n; pk = iota; k
// unit() feature columns drawn column by column from derive_seed(seed, "dim")
// (as make_dim draws features, benchgen.cpp:96-99), stored row-major; W =
// gen_linear(k, l, 7) (row-major k x l).
// ---- matrix / selection API (matrix.cpp:81-123, 198-255; laqops.cpp:65-121, 457-478)
SparseCsr make_csr(const int64_t* rp, const int64_t* ci, const double* v, int64_t rows, int64_t cols) {
  SparseCsr m;
  m.rows = rows;
  m.cols = cols;
  m.row_ptr.assign(rp, rp + rows + 1);
  const int64_t nnz = rp[rows];
  m.col_idx.assign(ci, ci + nnz);
  m.values.assign(v, v + nnz);
  return m;
}

int ref_spmm(const int64_t* a_rp, const int64_t* a_ci, const double* a_v, int64_t a_rows, int64_t a_cols,
             const int64_t* b_rp, const int64_t* b_ci, const double* b_v, int64_t b_rows, int64_t b_cols, int64_t cap,
             int64_t* c_rp, int64_t* c_ci, double* c_v, int64_t* nnz) {
  return guard([&] {
    const SparseCsr c = spmm(make_csr(a_rp, a_ci, a_v, a_rows, a_cols), make_csr(b_rp, b_ci, b_v, b_rows, b_cols));
    *nnz = c.nnz();
    if (c.nnz() > cap) throw CapacityError("output capacity");
    std::copy(c.row_ptr.begin(), c.row_ptr.end(), c_rp);
    std::copy(c.col_idx.begin(), c.col_idx.end(), c_ci);
    std::copy(c.values.begin(), c.values.end(), c_v);
  });
}

int ref_csr_from_coo(const int64_t* r, const int64_t* c, const double* v, int64_t nnz, int64_t rows, int64_t cols,
                     int64_t* rp) {
  return guard([&] {
    SparseCoo m;
    m.rows = rows;
    m.cols = cols;
    m.row_idx.assign(r, r + nnz);
    m.col_idx.assign(c, c + nnz);
    m.values.assign(v, v + nnz);
    const SparseCsr out = csr_from_coo(m);
    std::copy(out.row_ptr.begin(), out.row_ptr.end(), rp);
  });
}

int ref_coo_from_csr(const int64_t* rp, const int64_t* ci, const double* v, int64_t rows, int64_t cols, int64_t* r) {
  return guard([&] {
    const SparseCoo m = coo_from_csr(make_csr(rp, ci, v, rows, cols));
    std::copy(m.row_idx.begin(), m.row_idx.end(), r);
  });
}

int ref_sort_rows(const double* t, int64_t rows, int64_t cols, const int64_t* keys, const int32_t* desc, int32_t nk,
                  double* out) {
  return guard([&] {
    DenseMat m(rows, cols, std::vector<double>(t, t + rows * cols));
    std::vector<index_t> kc(keys, keys + nk);
    std::vector<ops::SortDir> d;
    for (int32_t k = 0; k < nk; ++k) d.push_back(desc[k] ? ops::SortDir::Desc : ops::SortDir::Asc);
    const DenseMat o = ops::sort_rows(m, kc, d);
    std::copy(o.data().begin(), o.data().end(), out);
  });
}

// build_selection_mask over an int64 (is_float = 0) or double column with a typed predicate.
int ref_selection_mask(const void* col, int is_float, int64_t n, int kind, int pred_float, int64_t ilo, int64_t ihi,
                       double flo, double fhi, const int64_t* iset, const double* fset, int64_t set_len,
                       uint8_t* out) {
  return guard([&] {
    auto make = [&]() -> Predicate {
      if (pred_float) {
        switch (kind) {
          case LAQ_PRED_LT: return Predicate::lt(flo);
          case LAQ_PRED_LE: return Predicate::le(flo);
          case LAQ_PRED_EQ: return Predicate::eq(flo);
          case LAQ_PRED_GE: return Predicate::ge(flo);
          case LAQ_PRED_GT: return Predicate::gt(flo);
          case LAQ_PRED_BETWEEN: return Predicate::between(flo, fhi);
          default: return Predicate::in_set(std::vector<double>(fset, fset + set_len));
        }
      }
      switch (kind) {
        case LAQ_PRED_LT: return Predicate::lt(ilo);
        case LAQ_PRED_LE: return Predicate::le(ilo);
        case LAQ_PRED_EQ: return Predicate::eq(ilo);
        case LAQ_PRED_GE: return Predicate::ge(ilo);
        case LAQ_PRED_GT: return Predicate::gt(ilo);
        case LAQ_PRED_BETWEEN: return Predicate::between(ilo, ihi);
        default: return Predicate::in_set(std::vector<std::int64_t>(iset, iset + set_len));
      }
    };
    const Predicate p = make();
    const ops::SelectionMask m =
        is_float ? ops::build_selection_mask(FloatColumn(static_cast<const double*>(col),
                                                          static_cast<const double*>(col) + n), p)
                 : ops::build_selection_mask(IntColumn(static_cast<const int64_t*>(col),
                                                       static_cast<const int64_t*>(col) + n), p);
    for (int64_t i = 0; i < n; ++i) out[i] = m.bits[i] ? 1 : 0;
  });
}

int ref_cfg1_inputs(int64_t n, int64_t dim_rows, int64_t k, int64_t l, uint64_t seed, int64_t* fk, int64_t* pk,
                    double* feats, double* w) {
  return guard([&] {
    Rng rf(derive_seed(seed, "lineorder"));
    for (int64_t i = 0; i < n; ++i) fk[i] = rf.range(0, dim_rows);
    for (int64_t i = 0; i < dim_rows; ++i) pk[i] = i;
    Rng rd(derive_seed(seed, "dim"));
    for (int64_t c = 0; c < k; ++c)
      for (int64_t r = 0; r < dim_rows; ++r) feats[r * k + c] = rd.unit();
    const ml::LinearOperator op = bench::gen_linear(k, l, 7);
    std::copy(op.mat.data().begin(), op.mat.data().end(), w);
  });
}

int ref_fused_pipeline(int n_links, const int64_t* const* fks, int64_t n, const int64_t* const* pks,
                       const int64_t* pk_rows, const double* const* feats, const int64_t* kj,
                       const double* L, int64_t l, double* out_y, int64_t* nnz, double* seconds) {
  return guard([&] {
    Schema fs;
    std::vector<Column> fc;
    std::vector<std::string> fnames;
    for (int j = 0; j < n_links; ++j) {
      fnames.push_back("f" + std::to_string(j));
      fs.columns.emplace_back(fnames.back(), ColKind::Key);
      fc.emplace_back(IntColumn(fks[j], fks[j] + n));
    }
    const Table fact(fs, std::move(fc));
    std::vector<Table> dims;
    for (int j = 0; j < n_links; ++j) dims.push_back(key_table(pks[j], pk_rows[j], "k"));
    std::vector<ops::DimJoinSpec> specs;
    for (int j = 0; j < n_links; ++j) specs.push_back({&dims[j], fnames[j], "k"});
    int64_t k = 0;
    for (int j = 0; j < n_links; ++j) k += kj[j];
    std::vector<DenseMat> dm;
    std::vector<ops::ColumnMap> maps;
    int64_t off = 0;
    for (int j = 0; j < n_links; ++j) {
      dm.emplace_back(pk_rows[j], kj[j], std::vector<double>(feats[j], feats[j] + pk_rows[j] * kj[j]));
      std::vector<std::pair<index_t, index_t>> mapping;
      for (int64_t c = 0; c < kj[j]; ++c) mapping.emplace_back(c, off + c);
      maps.push_back(ops::build_placement_map(kj[j], k, mapping));
      off += kj[j];
    }
    ml::LinearOperator op{DenseMat(k, l, std::vector<double>(L, L + k * l))};

    double t0 = now_s();
    const auto matches = ops::multiway_star_join(fact, specs);
    double t1 = now_s();
    std::vector<SparseCsr> imaps;
    for (const auto& mm : matches) imaps.push_back(csr_from_coo(mm.mat));
    double t2 = now_s();
    const auto f = fusion::prefuse_linear(dm, maps, op);
    double t3 = now_s();
    const DenseMat y = fusion::apply_fused_linear(imaps, f);
    double t4 = now_s();
    if (seconds) {
      seconds[0] = t1 - t0;
      seconds[1] = t2 - t1;
      seconds[2] = t3 - t2;
      seconds[3] = t4 - t3;
    }
    *nnz = y.rows();
    if (out_y) std::copy(y.data().begin(), y.data().end(), out_y);
  });
}

// ---- cost model (fusion.cpp:259-302) --------------------------------------
// ---- decision trees (mlops.cpp:188-280, fusion.cpp:39-168, benchgen.cpp:463-...) ----
namespace {
ml::TreeModel make_tree(int n_nodes, const int32_t* is_leaf, const int64_t* feature, const double* thr,
                        const int64_t* tchild, const int64_t* fchild, const int64_t* label) {
  ml::TreeModel t;
  for (int i = 0; i < n_nodes; ++i)
    t.nodes.push_back({is_leaf[i] != 0, feature[i], thr[i], tchild[i], fchild[i], label[i]});
  return t;
}
}  // namespace

// gen_tree -> node arrays (capacity cap); *n = node count.
int ref_gen_tree(int64_t k, int64_t p, int64_t leaves, uint64_t seed, int64_t cap, int32_t* is_leaf,
                 int64_t* feature, double* thr, int64_t* tchild, int64_t* fchild, int64_t* label, int64_t* n) {
  return guard([&] {
    const ml::TreeModel t = bench::gen_tree(k, p, leaves, seed);
    *n = static_cast<int64_t>(t.nodes.size());
    if (*n > cap) throw CapacityError("ref_gen_tree: capacity");
    for (size_t i = 0; i < t.nodes.size(); ++i) {
      const auto& nd = t.nodes[i];
      is_leaf[i] = nd.is_leaf;
      feature[i] = nd.feature;
      thr[i] = nd.threshold;
      tchild[i] = nd.true_child;
      fchild[i] = nd.false_child;
      label[i] = nd.label;
    }
  });
}

// compile_tree + predict_tree over T (rows x k).
int ref_predict_tree(int n_nodes, const int32_t* is_leaf, const int64_t* feature, const double* thr,
                     const int64_t* tchild, const int64_t* fchild, const int64_t* label, const double* T,
                     int64_t rows, int64_t k, int64_t* out) {
  return guard([&] {
    const ml::TreeLA m = ml::compile_tree(make_tree(n_nodes, is_leaf, feature, thr, tchild, fchild, label), k);
    const DenseMat t(rows, k, std::vector<double>(T, T + rows * k));
    const auto y = ml::predict_tree(t, m);
    std::copy(y.begin(), y.end(), out);
  });
}

// compile_tree -> partition_tree(feature_owner) -> prefuse_tree -> apply_fused_tree over
// row maps idx (m rows).  partials[j] receives r_j x leaves (may be NULL).
int ref_fused_tree(int n_nodes, const int32_t* is_leaf, const int64_t* feature, const double* thr,
                   const int64_t* tchild, const int64_t* fchild, const int64_t* label, int n_dims,
                   const double* const* dims, const int64_t* rows, const int64_t* cols,
                   const int64_t* const* placements, int64_t k, const int64_t* feature_owner,
                   const int64_t* const* idx, int64_t m, int64_t* out, double* const* partials) {
  return guard([&] {
    const ml::TreeLA t = ml::compile_tree(make_tree(n_nodes, is_leaf, feature, thr, tchild, fchild, label), k);
    StarMats s = make_mats(n_dims, dims, rows, cols, placements, k, idx, m);
    const auto parts = fusion::partition_tree(t, std::vector<index_t>(feature_owner, feature_owner + k), n_dims);
    const auto f = fusion::prefuse_tree(s.dims, s.maps, parts, t.path_score, t.labels);
    if (partials)
      for (int j = 0; j < n_dims; ++j)
        if (partials[j]) std::copy(f.partials[j].data().begin(), f.partials[j].data().end(), partials[j]);
    if (idx && out) {
      const auto y = fusion::apply_fused_tree(s.imaps, f);
      std::copy(y.begin(), y.end(), out);
    }
  });
}

int ref_speedup_ratio(int tree, int64_t i, int64_t k, int64_t l, int64_t p, const int64_t* dims,
                      int n, double* out) {
  return guard([&] {
    fusion::CostInputs c;
    c.target_rows = i;
    c.input_width = k;
    c.output_width = l;
    c.tree_features = p;
    c.dim_rows.assign(dims, dims + n);
    *out = tree ? fusion::speedup_ratio_tree(c) : fusion::speedup_ratio_linear(c);
  });
}

int ref_decide_fusion(double ratio, double threshold, int* out) {
  return guard([&] { *out = fusion::decide_fusion(ratio, threshold) ? 1 : 0; });
}

// ---- report helpers (report.cpp:90-146) -----------------------------------
uint64_t ref_checksum_rows(const double* data, int64_t rows, int64_t cols) {
  const DenseMat m(rows, cols, std::vector<double>(data, data + rows * cols));
  return cli::checksum_rows(m);
}

}  // extern "C"
