// configs[0] (fused join + linear predict, 1M-row fact x 10K-row dim, k=16,
// l=1) end to end through the reference's UNCHANGED C++ API with host
// std::vector buffers, served by the drop-in (B200 C-ABI underneath): the same
// call sequence as the reference's own pipeline (cli.cpp:279-346,
// ref_fused_pipeline in oracle/ref_capi.cpp) -- multiway_star_join ->
// csr_from_coo -> prefuse_linear -> apply_fused_linear.  Every call moves its
// inputs host->device and its outputs device->host, as a C++ caller of the
// reference API would see it.
//
//   dropin_bench <dir> [reps]
// <dir> holds fk.bin (int64 x n), pk.bin (int64 x r), feats.bin (f64 r x k),
// W.bin (f64 k x l) and meta.txt ("n r k l"); y.bin (f64 n x l) is written
// back for the caller's bit-exactness check.  Prints one JSON line of median
// per-stage seconds over `reps` timed repetitions (after 2 warm-ups).
//
//   dropin_bench --query <sf> <dial21> <dial31> [reps]
// SSB-style queries through cli::run_query_laq (cli.cpp:73-138) on the
// reference generator's data (bench::gen_star, Setting::Ssb, seed 42): Q2.1 and
// Q3.1 with the given dials (the query defs of benchgen.cpp:259-289).  Times
// the first call (H2D of the query's columns into the drop-in's device cache +
// the device run) and the cached calls after it, and checks every result
// against the reference's own run_query_oracle (cli.cpp:140-225) at tolerance 0.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "laq/benchgen.hpp"
#include "laq/cli.hpp"
#include "laq/fusion.hpp"
#include "laq/laqops.hpp"
#include "laq/matrix.hpp"
#include "laq/mlops.hpp"
#include "laq/predicate.hpp"
#include "laq/report.hpp"
#include "laq/storage.hpp"

using namespace laq;

template <class T>
static std::vector<T> load(const std::string& path, size_t n) {
  std::vector<T> v(n);
  std::ifstream f(path, std::ios::binary);
  f.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n * sizeof(T)));
  if (!f) throw std::runtime_error("short read: " + path);
  return v;
}

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

static int query_mode(int argc, char** argv) {
  if (argc < 5) return 2;
  bench::GenConfig cfg;
  cfg.setting = bench::Setting::Ssb;
  cfg.sf = std::atoi(argv[2]);
  cfg.seed = 42;
  cfg.max_bytes = std::int64_t{64} << 30;
  const int reps = argc > 5 ? std::atoi(argv[5]) : 5;
  double t0 = now_s();
  const StarSchema s = bench::gen_star(cfg);
  const double gen_s = now_s() - t0;
  const StarLink part{"lo_part", "part", "p_key"}, supp{"lo_supplier", "supplier", "s_key"},
      date{"lo_orderdate", "date", "d_key"};
  bench::QuerySpec q21;  // benchgen.cpp:259-266
  q21.id = "21";
  q21.group = bench::QueryGroup::G2;
  q21.joins = {part, supp, date};
  q21.filters = {{1, "s_region", Predicate::eq(std::int64_t{0})}, {0, "p_size", Predicate::lt(static_cast<std::int64_t>(std::atoll(argv[3])))}};
  q21.measure = "lo_revenue";
  q21.group_by = {{2, "d_year"}, {0, "p_brand"}};
  q21.order_by = true;
  bench::QuerySpec q31;  // benchgen.cpp:283-289
  q31.id = "31";
  q31.group = bench::QueryGroup::G3;
  q31.joins = {part, supp, date};
  q31.filters = {{2, "d_year", Predicate::between(std::int64_t{1992}, std::int64_t{1997})},
                 {1, "s_rank", Predicate::lt(static_cast<std::int64_t>(std::atoll(argv[4])))}};
  q31.measure = "lo_revenue";
  q31.group_by = {{1, "s_nation"}, {2, "d_year"}};
  q31.order_by = true;
  std::printf("{\"sf\": %d, \"fact_rows\": %lld, \"gen_s\": %.3f", cfg.sf,
              static_cast<long long>(s.fact().row_count()), gen_s);
  for (const auto* q : {&q21, &q31}) {
    t0 = now_s();
    const DenseMat first = cli::run_query_laq(s, *q);
    const double cold = now_s() - t0;
    std::vector<double> warm;
    DenseMat last;
    for (int i = 0; i < reps; ++i) {
      t0 = now_s();
      last = cli::run_query_laq(s, *q);
      warm.push_back(now_s() - t0);
    }
    t0 = now_s();
    const DenseMat want = cli::run_query_oracle(s, *q);
    const double oracle_s = now_s() - t0;
    const bool ok = cli::compare_matrices(first, want, 0.0).ok && cli::compare_matrices(last, want, 0.0).ok;
    std::printf(", \"Q%s\": {\"rows\": %lld, \"first_call_s\": %.6g, \"cached_call_s\": %.6g, "
                "\"reference_oracle_s\": %.6g, \"equal_to_reference_oracle\": %s}",
                q->id.c_str(), static_cast<long long>(first.rows()), cold, median(warm), oracle_s,
                ok ? "true" : "false");
  }
  std::printf("}\n");
  return 0;
}

// dropin_bench --pipeline <sf> [reps]: the reference's PipelineRunner (cli.cpp:246-378)
// on its acceptance dataset shape (S2, seed 9001, 64 features, linear model with
// 4 outputs): one-time prepare_joins + prefuse, then run_fused / run_nonfused
// repetitions; every result's checksum must equal run_oracle's.
static int pipeline_mode(int argc, char** argv) {
  if (argc < 3) return 2;
  bench::GenConfig cfg;
  cfg.setting = bench::Setting::S2;
  cfg.sf = std::atoi(argv[2]);
  cfg.seed = 9001;
  cfg.feature_width = 64;
  const int reps = argc > 3 ? std::atoi(argv[3]) : 5;
  const StarSchema s = bench::gen_star(cfg);
  const bench::FeatureLayout lay = bench::feature_layout(s);
  const ml::LinearOperator op = bench::gen_linear(lay.total, 4, 3);
  cli::PipelineRunner runner(s, nullptr, &op);
  cli::StageTimes st;
  double t0 = now_s();
  runner.prepare_joins(st);
  const double join_s = now_s() - t0;
  t0 = now_s();
  runner.prefuse(st);
  const double prefuse_s = now_s() - t0;
  std::vector<double> tf, tn;
  uint64_t cf = 0, cn = 0;
  for (int i = 0; i < reps + 1; ++i) {
    t0 = now_s();
    const cli::PipelineResult f = runner.run_fused(st);
    const double a = now_s() - t0;
    t0 = now_s();
    const cli::PipelineResult n = runner.run_nonfused(st);
    const double b = now_s() - t0;
    cf = f.checksum();
    cn = n.checksum();
    if (i > 0) tf.push_back(a), tn.push_back(b);
  }
  t0 = now_s();
  const uint64_t co = runner.run_oracle(st).checksum();
  const double oracle_s = now_s() - t0;
  std::printf("{\"sf\": %d, \"target_rows\": %lld, \"k\": %lld, \"l\": 4, \"prepare_joins_s\": %.6g, "
              "\"prefuse_s\": %.6g, \"run_fused_s\": %.6g, \"run_nonfused_s\": %.6g, \"run_oracle_s\": %.6g, "
              "\"checksum_fused\": \"%llu\", \"checksum_nonfused\": \"%llu\", \"checksum_oracle\": \"%llu\", "
              "\"fused_equals_oracle\": %s, \"nonfused_equals_oracle\": %s}\n",
              cfg.sf, static_cast<long long>(runner.target_rows()), static_cast<long long>(lay.total), join_s,
              prefuse_s, median(tf), median(tn), oracle_s, static_cast<unsigned long long>(cf),
              static_cast<unsigned long long>(cn), static_cast<unsigned long long>(co), cf == co ? "true" : "false",
              cn == co ? "true" : "false");
  return 0;
}

int main(int argc, char** argv) {
  if (argc >= 2 && std::string(argv[1]) == "--query") return query_mode(argc, argv);
  if (argc >= 2 && std::string(argv[1]) == "--pipeline") return pipeline_mode(argc, argv);
  if (argc < 2) {
    std::fprintf(stderr, "usage: dropin_bench <dir> [reps]\n");
    return 2;
  }
  const std::string dir = argv[1];
  const int reps = argc > 2 ? std::atoi(argv[2]) : 10;
  long long n = 0, r = 0, k = 0, l = 0;
  {
    std::ifstream m(dir + "/meta.txt");
    m >> n >> r >> k >> l;
  }
  Schema fs;
  fs.columns.emplace_back("fk", ColKind::Key);
  std::vector<Column> fc;
  fc.emplace_back(load<std::int64_t>(dir + "/fk.bin", static_cast<size_t>(n)));
  const Table fact(fs, std::move(fc));
  Schema ds;
  ds.columns.emplace_back("pk", ColKind::Key);
  std::vector<Column> dc;
  dc.emplace_back(load<std::int64_t>(dir + "/pk.bin", static_cast<size_t>(r)));
  const Table dim(ds, std::move(dc));
  const std::vector<ops::DimJoinSpec> specs{{&dim, "fk", "pk"}};
  const std::vector<DenseMat> dm{DenseMat(r, k, load<double>(dir + "/feats.bin", static_cast<size_t>(r * k)))};
  std::vector<std::pair<index_t, index_t>> mapping;
  for (long long c = 0; c < k; ++c) mapping.emplace_back(c, c);
  const std::vector<ops::ColumnMap> maps{ops::build_placement_map(k, k, mapping)};
  const ml::LinearOperator op{DenseMat(k, l, load<double>(dir + "/W.bin", static_cast<size_t>(k * l)))};

  std::vector<double> t_join, t_csr, t_pre, t_apply;
  DenseMat y;
  for (int it = 0; it < reps + 2; ++it) {
    const double t0 = now_s();
    const auto matches = ops::multiway_star_join(fact, specs);
    const double t1 = now_s();
    std::vector<SparseCsr> imaps;
    for (const auto& mm : matches) imaps.push_back(csr_from_coo(mm.mat));
    const double t2 = now_s();
    const auto f = fusion::prefuse_linear(dm, maps, op);
    const double t3 = now_s();
    y = fusion::apply_fused_linear(imaps, f);
    const double t4 = now_s();
    if (it >= 2) {
      t_join.push_back(t1 - t0);
      t_csr.push_back(t2 - t1);
      t_pre.push_back(t3 - t2);
      t_apply.push_back(t4 - t3);
    }
  }
  {
    std::ofstream o(dir + "/y.bin", std::ios::binary);
    o.write(reinterpret_cast<const char*>(y.data().data()), static_cast<std::streamsize>(y.data().size() * 8));
  }
  const double call = median(t_join) + median(t_csr) + median(t_apply);
  std::printf(
      "{\"rows\": %lld, \"nnz\": %lld, \"reps\": %d, \"multiway_star_join_s\": %.6g, \"csr_from_coo_s\": %.6g, "
      "\"prefuse_linear_s\": %.6g, \"apply_fused_linear_s\": %.6g, \"join_csr_apply_s\": %.6g, "
      "\"rows_per_s\": %.6g}\n",
      n, static_cast<long long>(y.rows()), reps, median(t_join), median(t_csr), median(t_pre), median(t_apply), call,
      static_cast<double>(n) / call);
  return 0;
}
