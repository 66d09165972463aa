// C++ drop-in contract details checked against the reference library
// (oracle/_ref/libmgr_ref.so, test infrastructure):
//   * PassStats of decompose AND recompose (acceptance criterion 9,
//     acceptance.cpp:336-374; refactor.hpp:159-199, 223-421) equal the
//     reference engine's counters record for record;
//   * weighted_l2_norm (grid.hpp:198-244) bit-identical;
//   * RefactorOptions::levels = 0 -> InvalidLevel (grid.cpp:99-102);
//   * the per-thread plan cache is bounded (LRU) and results stay exact;
//   * embarrassing_decompose with the reference's signature (devices from
//     the runtime), grouped_decompose running its groups concurrently;
//   * CommReport::to_json byte-identical to the reference's formatter, and a
//     caller shaped like mgrf.cpp:146-158 compiles and writes a report with
//     idle records;
//   * write_refactored rejects a class prefix / mis-sized class instead of
//     over-reading (MissingClass / ShapeError).
// Build + run: tests/test_cpp_shim.py.  Prints "dropin ok" on success.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>

#include "mgr_b200/parallel.hpp"
#include "mgr_b200/pipeline.hpp"

extern "C" {
int mgrref_decompose_f64(int, const uint64_t *, const double *, int, const double *,
                         double *, int *);
int mgrref_pass_stats_f64(int, const uint64_t *, const double *, int, const double *, int,
                          uint64_t *, int, int *);
double mgrref_weighted_l2_norm_f64(int, const uint64_t *, const double *, const double *);
int mgrref_comm_report_json(int, int, uint64_t, int, const char *const *, const uint64_t *,
                            const double *, int, const uint64_t *, char *, uint64_t);
}

#define CHECK(c)                                                               \
  do {                                                                         \
    if (!(c)) {                                                                \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);\
      std::exit(1);                                                            \
    }                                                                          \
  } while (0)

static std::vector<std::vector<double>> rand_coords(const mgr::Shape &shape, unsigned seed) {
  std::mt19937 gen(seed);
  std::uniform_real_distribution<double> S(0.1, 1.0);
  std::vector<std::vector<double>> coords;
  for (std::size_t n : shape) {
    std::vector<double> c(n);
    double acc = 0;
    for (auto &x : c)
      x = (acc += S(gen));
    coords.push_back(c);
  }
  return coords;
}

static std::vector<double> rand_values(std::size_t n, unsigned seed) {
  std::mt19937 gen(seed);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  std::vector<double> v(n);
  for (auto &x : v)
    x = U(gen);
  return v;
}

static std::vector<double> flat_coords(const std::vector<std::vector<double>> &c) {
  std::vector<double> f;
  for (const auto &x : c)
    f.insert(f.end(), x.begin(), x.end());
  return f;
}

static void check_stats_equal(const mgr::PassStats &st, const std::vector<uint64_t> &ref,
                              int nrec, std::size_t nd) {
  CHECK(st.levels.size() == std::size_t(nrec));
  const std::size_t w = 8 + 4 * nd;
  for (int i = 0; i < nrec; ++i) {
    const auto &lv = st.levels[i];
    const uint64_t *o = ref.data() + i * w;
    CHECK(lv.level == o[0] && lv.level_elements == o[1]);
    CHECK(lv.coefficient.in == o[2] && lv.coefficient.out == o[3]);
    CHECK(lv.fused_copy.in == o[4] && lv.fused_copy.out == o[5]);
    CHECK(lv.masstrans.size() == nd && lv.solve.size() == nd);
    for (std::size_t d = 0; d < nd; ++d) {
      CHECK(lv.masstrans[d].in == o[6 + 2 * d] && lv.masstrans[d].out == o[7 + 2 * d]);
      CHECK(lv.solve[d].in == o[6 + 2 * nd + 2 * d] &&
            lv.solve[d].out == o[7 + 2 * nd + 2 * d]);
    }
    CHECK(lv.apply.in == o[6 + 4 * nd] && lv.apply.out == o[7 + 4 * nd]);
  }
}

static void pass_stats_case(const mgr::Shape &shape, bool nonuniform, int cap) {
  const auto coords = nonuniform ? rand_coords(shape, 11) : std::vector<std::vector<double>>{};
  const auto v = rand_values(mgr::num_elements(shape), 9000);
  const auto g = mgr::make_grid<double>(shape, v, coords);
  mgr::PassStats st;
  mgr::RefactorOptions opt;
  if (cap)
    opt.levels = std::size_t(cap);
  opt.stats = &st;
  const auto r = mgr::decompose(g, opt);
  std::vector<uint64_t> sh(shape.begin(), shape.end());
  const auto cf = flat_coords(g.coords);
  const std::size_t nd = shape.size();
  std::vector<uint64_t> ref(64 * (8 + 4 * nd));
  int n = 0;
  CHECK(mgrref_pass_stats_f64(int(nd), sh.data(), cf.data(), cap, v.data(), 0, ref.data(), 64,
                              &n) == 0);
  check_stats_equal(st, ref, n, nd);
  // recompose appends (coarsest first) to the same stats object
  (void)mgr::recompose(r, r.levels, opt);
  CHECK(mgrref_pass_stats_f64(int(nd), sh.data(), cf.data(), cap, v.data(), 1, ref.data(), 64,
                              &n) == 0);
  check_stats_equal(st, ref, n, nd);
  CHECK(st.levels.size() == 2 * r.levels);
}

// A caller shaped like the reference CLI's refactor command (mgrf.cpp:146-165).
template <typename Real>
std::string cli_like_refactor(const mgr::TensorGrid<Real> &grid, int workers,
                              std::optional<std::size_t> levels, const std::string &stats_path) {
  using namespace mgr;
  RefactoredData<Real> r;
  PassStats passes;
  if (workers > 1) {
    CoopOptions opt;
    if (levels)
      opt.levels = levels;
    opt.scheme = PartitionScheme::block;
    CommReport report;
    opt.report = &report;
    r = cooperative_decompose(grid, workers, opt);
    if (!stats_path.empty()) {
      std::ofstream out(stats_path, std::ios::trunc);
      out << report.to_json() << "\n";
    }
    return report.to_json();
  }
  RefactorOptions opt;
  if (levels)
    opt.levels = levels;
  opt.stats = &passes;
  r = decompose(grid, opt);
  return std::to_string(passes.levels.size());
}

int main(int argc, char **argv) {
  const std::string tmp = argc > 1 ? argv[1] : "/tmp";
  // ---- criterion 9 (acceptance.cpp:336-374) + recompose accounting
  pass_stats_case({17, 17, 17}, false, 0);
  pass_stats_case({12, 10, 9}, false, 0);
  pass_stats_case({33, 17}, true, 0);
  pass_stats_case({65}, false, 3);
  pass_stats_case({9, 5, 3, 6}, true, 0);
  // ---- weighted_l2_norm bit-identical (3-D non-uniform, 2-D, 1-D)
  for (const mgr::Shape &shape : {mgr::Shape{9, 7, 5}, mgr::Shape{33, 12}, mgr::Shape{17}}) {
    const auto coords = rand_coords(shape, 5);
    const auto v = rand_values(mgr::num_elements(shape), 6);
    const auto g = mgr::make_grid<double>(shape, v, coords);
    std::vector<uint64_t> sh(shape.begin(), shape.end());
    const auto cf = flat_coords(coords);
    const double ref = mgrref_weighted_l2_norm_f64(int(shape.size()), sh.data(), cf.data(),
                                                   v.data());
    const double got = mgr::weighted_l2_norm(g);
    CHECK(std::memcmp(&ref, &got, sizeof(double)) == 0);
  }
  // ---- levels = 0 is InvalidLevel (grid.cpp:99-102), in both APIs
  {
    const auto g = mgr::make_grid<double>({9, 9}, rand_values(81, 1));
    mgr::RefactorOptions opt;
    opt.levels = 0;
    try {
      (void)mgr::decompose(g, opt);
      CHECK(false);
    } catch (const mgr::InvalidLevel &e) {
      CHECK(std::string(e.what()) == "level count must be at least 1");
    }
    mgr::CoopOptions co;
    co.levels = 0;
    const auto g3 = mgr::make_grid<double>({9, 9, 9}, rand_values(729, 2));
    try {
      (void)mgr::cooperative_decompose(g3, 2, co);
      CHECK(false);
    } catch (const mgr::InvalidLevel &) {
    }
    // a huge cap is the full depth, not a wrapped negative
    opt.levels = std::size_t(1) << 40;
    CHECK(mgr::decompose(g, opt).levels == 3);
  }
  // ---- bounded plan cache: 2 plans, 5 geometries cycled twice, exact results
  {
    const std::size_t old = mgr::set_plan_cache_capacity(2);
    for (int rep = 0; rep < 2; ++rep)
      for (std::size_t n : {9, 17, 33, 12, 20}) {
        const mgr::Shape shape{n, 9};
        const auto v = rand_values(n * 9, unsigned(n));
        const auto r = mgr::decompose(mgr::make_grid<double>(shape, v));
        std::vector<uint64_t> sh(shape.begin(), shape.end());
        const auto cf = flat_coords({mgr::uniform_coords(n), mgr::uniform_coords(9)});
        std::vector<double> ref(v.size());
        int L = 0;
        CHECK(mgrref_decompose_f64(2, sh.data(), cf.data(), 0, v.data(), ref.data(), &L) == 0);
        std::size_t off = 0;
        for (const auto &c : r.classes) {
          CHECK(std::memcmp(c.data(), ref.data() + off, c.size() * sizeof(double)) == 0);
          off += c.size();
        }
      }
    mgr::release_plans();
    mgr::set_plan_cache_capacity(old);
  }
  // ---- embarrassing_decompose (reference signature) / grouped_decompose
  {
    std::vector<mgr::TensorGrid<double>> blocks;
    for (unsigned i = 0; i < 5; ++i)
      blocks.push_back(mgr::make_grid<double>({17, 9, 9}, rand_values(17 * 81, 100 + i)));
    mgr::RefactorOptions ro;
    const auto e = mgr::embarrassing_decompose(blocks, 4, ro);
    const auto g = mgr::grouped_decompose(blocks, 2, 2, mgr::PartitionScheme::block);
    for (std::size_t i = 0; i < blocks.size(); ++i) {
      const auto one = mgr::decompose(blocks[i]);
      CHECK(e[i].classes == one.classes);
      CHECK(g[i].classes == one.classes);
    }
  }
  // ---- CommReport::to_json: byte-identical formatter
  {
    mgr::CommReport rep;
    rep.workers = 3;
    rep.scheme = mgr::PartitionScheme::shifted_round_robin;
    rep.total_grid_elements = 35937;
    rep.phases["device"] = {4, 12345, 7, 0.125};
    rep.phases["halo"] = {2, 99, 0, 1.5e-05};
    rep.idle.push_back({5, 2, {2, 2, 2}});
    rep.idle.push_back({4, 2, {2, 1}});
    const char *names[] = {"device", "halo"};
    const uint64_t counts[] = {4, 12345, 7, 2, 99, 0};
    const double secs[] = {0.125, 1.5e-05};
    const uint64_t idle[] = {5, 2, 3, 2, 2, 2, 4, 2, 2, 2, 1};
    char buf[4096];
    CHECK(mgrref_comm_report_json(3, 1, 35937, 2, names, counts, secs, 2, idle, buf,
                                  sizeof(buf)) == 0);
    CHECK(rep.to_json() == std::string(buf));
    // the CLI-shaped caller: a real cooperative run fills phases and idle
    const auto grid = mgr::make_grid<double>({33, 33, 33}, rand_values(33 * 33 * 33, 77));
    const std::string path = tmp + "/coop_stats.json";
    const std::string j = cli_like_refactor(grid, 2, std::nullopt, path);
    CHECK(j.find("\"workers\":2") != std::string::npos);
    CHECK(j.find("\"idle\":[{\"level\":5,\"dim\":2,\"idle_per_stage\":[1,1]}") !=
          std::string::npos);
    std::ifstream in(path);
    std::stringstream ss;
    ss << in.rdbuf();
    CHECK(ss.str() == j + "\n");
    CHECK(cli_like_refactor(grid, 1, std::size_t(2), "") == "2");
  }
  // ---- write_refactored: prefix / mis-sized classes are rejected
  {
    const auto g = mgr::make_grid<double>({17, 9}, rand_values(153, 3));
    auto r = mgr::decompose(g);
    auto cut = r;
    cut.classes.resize(2);
    try {
      mgr::write_refactored(cut, tmp + "/cut.mgrf");
      CHECK(false);
    } catch (const mgr::MissingClass &) {
    }
    auto bad = r;
    bad.classes[1].pop_back();
    try {
      mgr::write_refactored(bad, tmp + "/bad.mgrf");
      CHECK(false);
    } catch (const mgr::ShapeError &) {
    }
    CHECK(mgr::write_refactored(r, tmp + "/ok.mgrf") > 0);
  }
  std::printf("dropin ok\n");
  return 0;
}
