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
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "laq/fusion.hpp"
#include "laq/laqops.hpp"
#include "laq/matrix.hpp"
#include "laq/mlops.hpp"
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

int main(int argc, char** argv) {
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
