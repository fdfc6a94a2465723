// Extra device checks of the drop-in that the reference's own suites do not
// exercise, run through the reference's UNCHANGED API and compared with the
// reference's own scalar oracle (run_query_oracle, cli.cpp:140-225, linked
// unmodified) at tolerance 0:
//   * run_query_laq's general device path (float measures, float predicates,
//     integers outside int32, duplicate keys hidden by dimension filters) and
//     its fast path with the per-StarSchema device cache (incl. in-place edits);
//   * the planner-driven PipelineRunner (run_auto, include/laq_dropin.hpp).
// Prints "[PASS] ..." / "[FAIL] ..." lines; exit status 1 on any failure.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "laq/benchgen.hpp"
#include "laq/cli.hpp"
#include "laq/oracle.hpp"
#include "laq/report.hpp"
#include "laq_dropin.hpp"

using namespace laq;

static int g_fail = 0;

static void report(const std::string& name, bool ok, const std::string& detail = "") {
  std::printf("[%s] %s%s%s\n", ok ? "PASS" : "FAIL", name.c_str(), detail.empty() ? "" : ": ", detail.c_str());
  if (!ok) ++g_fail;
}

static bool same(const DenseMat& a, const DenseMat& b, std::string* why) {
  const cli::CompareResult r = cli::compare_matrices(a, b, 0.0);
  if (!r.ok) *why = r.diff;
  return r.ok;
}

static DenseMat oracle_float_measure(const StarSchema& s, const bench::QuerySpec& q);

static void check_query(const StarSchema& s, const bench::QuerySpec& q, const std::string& name) {
  std::string why;
  const bool float_measure = s.fact().schema().kind(s.fact().schema().index_of(q.measure)) == ColKind::Float;
  const DenseMat want = float_measure ? oracle_float_measure(s, q) : cli::run_query_oracle(s, q);
  setenv("LAQ_DROPIN_PATH", "", 1);
  const DenseMat fast = cli::run_query_laq(s, q);
  setenv("LAQ_DROPIN_PATH", "general", 1);
  const DenseMat gen = cli::run_query_laq(s, q);
  setenv("LAQ_DROPIN_PATH", "", 1);
  bool ok = same(fast, want, &why);
  report(name + " (default path)", ok, why);
  ok = same(gen, want, &why);
  report(name + " (general device path)", ok, why);
}

// Expected result for a FLOAT measure.  The reference's scalar oracle reads the
// measure with Table::ints (cli.cpp:194-196), so it cannot check these; the
// reference's run_query_laq reads it through to_matrix (cli.cpp:96-99), i.e.
// as doubles, summed per group in ascending fact-row order (groupby_sum_multi,
// laqops.cpp:415-455; the plain sum is dense_matmul's sequential loop).  Same
// scalar filter + oracle::star_join + oracle::hash_aggregate as the oracle,
// with the measure read as doubles.
static DenseMat oracle_float_measure(const StarSchema& s, const bench::QuerySpec& q) {
  auto filter = [&](const Table& t, int target) {
    std::vector<char> keep(static_cast<size_t>(t.row_count()), 1);
    for (const bench::FilterSpec& f : q.filters) {
      if (f.target != target) continue;
      const index_t c = t.schema().index_of(f.column);
      for (index_t r = 0; r < t.row_count(); ++r)
        if (keep[r]) keep[r] = t.schema().kind(c) == ColKind::Float ? f.pred.matches(t.floats(c)[r])
                                                                     : f.pred.matches(t.ints(c)[r]);
    }
    std::vector<Column> cols;
    for (index_t c = 0; c < t.col_count(); ++c) {
      if (std::holds_alternative<IntColumn>(t.column(c))) {
        IntColumn d;
        for (size_t r = 0; r < keep.size(); ++r) if (keep[r]) d.push_back(t.ints(c)[r]);
        cols.emplace_back(std::move(d));
      } else {
        FloatColumn d;
        for (size_t r = 0; r < keep.size(); ++r) if (keep[r]) d.push_back(t.floats(c)[r]);
        cols.emplace_back(std::move(d));
      }
    }
    return Table(t.schema(), std::move(cols));
  };
  const Table fact = filter(s.fact(), -1);
  std::vector<Table> dims;
  for (size_t j = 0; j < q.joins.size(); ++j) dims.push_back(filter(s.dim(q.joins[j].dim_name), static_cast<int>(j)));
  std::vector<oracle::DimRef> refs;
  for (size_t j = 0; j < q.joins.size(); ++j) refs.push_back({&dims[j], q.joins[j].fact_fk, q.joins[j].dim_pk});
  const oracle::StarMatch m = oracle::star_join(fact, refs);
  const FloatColumn& mv = fact.floats(q.measure);
  std::vector<double> vals;
  for (index_t r : m.fact_rows) vals.push_back(mv[r]);
  if (q.group_by.empty()) {
    double sum = 0;
    for (double v : vals) sum += v;
    return DenseMat(1, 1, {sum});
  }
  std::vector<IntColumn> gcols;
  for (const bench::GroupRef& g : q.group_by) {
    IntColumn col;
    const IntColumn& src = g.target < 0 ? fact.ints(g.column) : dims[g.target].ints(g.column);
    for (size_t i = 0; i < m.fact_rows.size(); ++i) col.push_back(src[g.target < 0 ? m.fact_rows[i] : m.dim_rows[g.target][i]]);
    gcols.push_back(std::move(col));
  }
  const auto agg = oracle::hash_aggregate(gcols, vals);
  DenseMat out(static_cast<index_t>(agg.size()), static_cast<index_t>(q.group_by.size()) + 1);
  for (size_t r = 0; r < agg.size(); ++r) {
    for (size_t c = 0; c < agg[r].keys.size(); ++c) out(static_cast<index_t>(r), static_cast<index_t>(c)) = static_cast<double>(agg[r].keys[c]);
    out(static_cast<index_t>(r), static_cast<index_t>(q.group_by.size())) = agg[r].sum;
  }
  return out;
}

// A star with extra fact columns: a float measure and 64-bit integers.
static StarSchema widened(const StarSchema& s) {
  const Table& f = s.fact();
  Schema sch = f.schema();
  std::vector<Column> cols;
  for (index_t c = 0; c < f.col_count(); ++c) cols.push_back(f.column(c));
  const IntColumn& rev = f.ints("lo_revenue");
  FloatColumn price(rev.size());
  IntColumn big(rev.size()), bigkey(rev.size());
  for (size_t i = 0; i < rev.size(); ++i) {
    price[i] = static_cast<double>(rev[i]) * 1.37 + 0.1 * static_cast<double>(i % 7);
    big[i] = rev[i] * (std::int64_t{1} << 40) + static_cast<std::int64_t>(i);
    bigkey[i] = (rev[i] % 5) * (std::int64_t{1} << 33);
  }
  sch.columns.push_back({"lo_price", ColKind::Float});
  cols.emplace_back(price);
  sch.columns.push_back({"lo_big", ColKind::Int});
  cols.emplace_back(big);
  sch.columns.push_back({"lo_bigkey", ColKind::Int});
  cols.emplace_back(bigkey);
  return StarSchema(Table(sch, std::move(cols)), s.dims(), s.links());
}

int main() {
  bench::GenConfig cfg;
  cfg.setting = bench::Setting::S2;
  cfg.sf = 2;
  cfg.seed = 42;
  cfg.feature_width = 6;
  const StarSchema base = bench::gen_star(cfg);
  const StarSchema s = widened(base);

  // 1. The workload's own queries (G1-G4, the reference tuner's dials).
  for (int g = 1; g <= 4; ++g)
    for (const bench::QuerySpec& q : bench::gen_queries(s, static_cast<bench::QueryGroup>(g)))
      check_query(s, q, "workload Q" + q.id);

  const StarLink part{"lo_part", "part", "p_key"}, supp{"lo_supplier", "supplier", "s_key"},
      date{"lo_orderdate", "date", "d_key"};
  // 2. Float measure, grouped and plain.
  {
    bench::QuerySpec q;
    q.id = "fm";
    q.joins = {part, date};
    q.filters = {{1, "d_year", Predicate::between(std::int64_t{1993}, std::int64_t{1996})}};
    q.measure = "lo_price";
    q.group_by = {{1, "d_year"}, {0, "p_brand"}};
    q.order_by = true;
    check_query(s, q, "float measure, group by (d_year, p_brand)");
    q.group_by.clear();
    check_query(s, q, "float measure, plain sum (sequential fp64)");
  }
  // 3. Float predicates on dimension feature columns, InSet and Between.
  {
    bench::QuerySpec q;
    q.id = "fp";
    q.joins = {part, supp};
    q.filters = {{0, "p_f0", Predicate::lt(0.5)}, {1, "s_f0", Predicate::between(0.2, 0.9)},
                 {-1, "lo_quantity", Predicate::in_set(std::vector<std::int64_t>{3, 7, 11, 40})}};
    q.measure = "lo_revenue";
    q.group_by = {{1, "s_nation"}};
    check_query(s, q, "float predicates + fact InSet");
  }
  // 4. Integers outside int32: measure and fact group column.
  {
    bench::QuerySpec q;
    q.id = "wide";
    q.joins = {date};
    q.filters = {{0, "d_month", Predicate::le(std::int64_t{6})}};
    q.measure = "lo_big";
    q.group_by = {{-1, "lo_bigkey"}, {0, "d_year"}};
    q.order_by = true;
    check_query(s, q, "int64 measure + 2^33-spaced fact group keys");
  }
  // 5. Duplicate dimension keys that the dimension filter removes.
  {
    const Table& d = s.dim("supplier");
    Schema sch = d.schema();
    std::vector<Column> cols;
    for (index_t c = 0; c < d.col_count(); ++c) cols.push_back(d.column(c));
    IntColumn keys = d.ints("s_key");
    IntColumn region = d.ints("s_region");
    keys.push_back(keys[0]);  // a duplicate of key 0 ...
    region.push_back(99);     // ... in a row the filter drops
    for (index_t c = 0; c < d.col_count(); ++c) {
      if (sch.name(c) == "s_key") cols[c] = keys;
      else if (sch.name(c) == "s_region") cols[c] = region;
      else if (std::holds_alternative<IntColumn>(cols[c])) std::get<IntColumn>(cols[c]).push_back(0);
      else std::get<FloatColumn>(cols[c]).push_back(0.0);
    }
    std::vector<std::pair<std::string, Table>> dims;
    for (const auto& [n, t] : s.dims()) dims.emplace_back(n, n == "supplier" ? Table(sch, cols) : t);
    std::vector<StarLink> links;  // StarSchema rejects duplicate pks on its own links (storage.cpp:200-213)
    for (const StarLink& l : s.links())
      if (l.dim_name != "supplier") links.push_back(l);
    const StarSchema s2(s.fact(), dims, links);
    bench::QuerySpec q;
    q.id = "dup";
    q.joins = {supp};
    q.filters = {{0, "s_region", Predicate::lt(std::int64_t{5})}};
    q.measure = "lo_revenue";
    q.group_by = {{0, "s_region"}};
    check_query(s2, q, "duplicate pk filtered out");
  }
  // 6. The device cache sees an in-place edit of a cached column.
  {
    StarSchema s3 = widened(base);
    bench::QuerySpec q = bench::gen_queries(s3, bench::QueryGroup::G2)[0];
    const DenseMat a = cli::run_query_laq(s3, q);
    IntColumn& rev = const_cast<IntColumn&>(s3.fact().ints("lo_revenue"));
    rev[0] += 12345;  // element 0 is always fingerprinted
    std::string why;
    const DenseMat b = cli::run_query_laq(s3, q);
    report("cache: in-place edit of a cached column is seen", same(b, cli::run_query_oracle(s3, q), &why) && !(a == b),
           why);
  }
  // 7. Planner-driven pipeline: run_auto runs the plan the cost model picks.
  {
    bench::GenConfig pc;
    pc.setting = bench::Setting::S2;
    pc.sf = 8;
    pc.seed = 9001;
    pc.feature_width = 64;
    const StarSchema ps = bench::gen_star(pc);
    for (index_t l : {4, 512}) {
      const ml::LinearOperator op = bench::gen_linear(64, l, 3);
      cli::PipelineRunner r(ps, nullptr, &op);
      cli::StageTimes st;
      cli::PlanChoice choice;
      const cli::PipelineResult got = cli::run_auto(r, st, 1.0, &choice);
      fusion::CostInputs c;
      c.target_rows = r.target_rows();
      c.input_width = 64;
      c.output_width = l;
      c.tree_features = 64;
      for (const std::string& n : r.layout().dim_names) c.dim_rows.push_back(ps.dim(n).row_count());
      const double ratio = fusion::speedup_ratio_linear(c);
      const cli::PipelineResult want = fusion::decide_fusion(ratio) ? r.run_fused(st) : r.run_nonfused(st);
      const cli::PipelineResult other = fusion::decide_fusion(ratio) ? r.run_nonfused(st) : r.run_fused(st);
      std::string why;
      const bool ok = choice.ratio == ratio && choice.fused == fusion::decide_fusion(ratio) &&
                      got.values == want.values && cli::compare_matrices(other.values, want.values, 1e-9).ok;
      report("run_auto l=" + std::to_string(l) + " picks " + (choice.fused ? "fused" : "non-fused") +
                 " (ratio " + std::to_string(ratio) + ")", ok);
    }
  }
  std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "OK", g_fail);
  return g_fail ? 1 : 0;
}
