// C++ drop-in check: code written against the reference's API
// (mgr::make_grid / decompose / recompose / recompose_with_report /
// embarrassing_decompose, refactor.hpp:462-534) compiled against
// include/mgr_b200/refactor.hpp, results compared bit-for-bit with the
// reference library itself (oracle/_ref/libmgr_ref.so, C harness
// oracle/ref_harness.cpp -- test infrastructure).
//
// Build + run: tests/test_cpp_shim.py.  Prints "shim ok" on success.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "mgr_b200/refactor.hpp"

extern "C" {
int mgrref_decompose_f64(int, const uint64_t *, const double *, int, const double *,
                         double *, int *);
int mgrref_decompose_f32(int, const uint64_t *, const double *, int, const float *,
                         float *, int *);
int mgrref_spatiotemporal_f64(int, const uint64_t *, const double *, int, const double *,
                              const double *, double *, int *);
}

#define CHECK(c)                                                               \
  do {                                                                         \
    if (!(c)) {                                                                \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);\
      std::exit(1);                                                            \
    }                                                                          \
  } while (0)

template <typename Real>
static void check_case(const mgr::Shape &shape, bool nonuniform, unsigned seed) {
  std::mt19937 gen(seed);
  std::uniform_real_distribution<double> U(0.0, 1.0), S(0.1, 1.0);
  std::vector<std::vector<double>> coords;
  if (nonuniform)
    for (std::size_t n : shape) {
      std::vector<double> c(n);
      double acc = 0;
      for (auto &x : c)
        x = (acc += S(gen));
      coords.push_back(c);
    }
  std::vector<Real> v(mgr::num_elements(shape));
  for (auto &x : v)
    x = Real(U(gen));
  const auto g = mgr::make_grid<Real>(shape, v, coords);
  const auto r = mgr::decompose(g);
  // reference on the same inputs
  std::vector<uint64_t> sh(shape.begin(), shape.end());
  std::vector<double> cflat;
  for (const auto &c : g.coords)
    cflat.insert(cflat.end(), c.begin(), c.end());
  std::vector<Real> ref(v.size());
  int L = 0;
  int st;
  if constexpr (sizeof(Real) == 8)
    st = mgrref_decompose_f64(int(shape.size()), sh.data(), cflat.data(), 0, v.data(),
                              ref.data(), &L);
  else
    st = mgrref_decompose_f32(int(shape.size()), sh.data(), cflat.data(), 0, v.data(),
                              ref.data(), &L);
  CHECK(st == 0);
  CHECK(std::size_t(L) == r.levels);
  std::size_t off = 0;
  for (const auto &c : r.classes) {
    CHECK(std::memcmp(c.data(), ref.data() + off, c.size() * sizeof(Real)) == 0);
    off += c.size();
  }
  CHECK(off == v.size());
  const auto back = mgr::recompose(r, r.levels);
  double err = 0;
  for (std::size_t i = 0; i < v.size(); ++i)
    err = std::max(err, std::abs(double(back.values[i]) - double(v[i])));
  CHECK(err <= (sizeof(Real) == 8 ? 1e-12 : 1e-5) * mgr::value_range(g));
  auto [rec0, rep] = mgr::recompose_with_report(r, 0, &g);
  CHECK(rep.classes_used == 0 && rep.max_abs_error > 0);
}

int main() {
  check_case<double>({33, 17, 9}, false, 1);
  check_case<float>({65, 40}, true, 2);
  check_case<double>({129}, true, 3);
  check_case<float>({12, 10, 9}, false, 4);
  check_case<double>({9, 5, 3, 6}, true, 5); // 4-D grids
  check_case<float>({17, 9, 5, 3}, false, 6);
  // decompose_spatiotemporal (refactor.hpp:536-567) against the reference's own
  {
    const mgr::Shape sh{9, 5, 5};
    const int T = 5;
    std::vector<mgr::TensorGrid<double>> snaps;
    std::vector<double> all, tc;
    for (int t = 0; t < T; ++t) {
      std::vector<double> v(9 * 5 * 5);
      for (std::size_t k = 0; k < v.size(); ++k)
        v[k] = std::cos(0.05 * double(k) + 0.3 * t);
      all.insert(all.end(), v.begin(), v.end());
      snaps.push_back(mgr::make_grid<double>(sh, v));
      tc.push_back(0.5 * t + 0.1 * t * t);
    }
    const auto r = mgr::decompose_spatiotemporal(snaps, tc);
    std::vector<uint64_t> s64(sh.begin(), sh.end());
    std::vector<double> ref(all.size());
    int L = 0;
    CHECK(mgrref_spatiotemporal_f64(3, s64.data(), nullptr, T, tc.data(), all.data(),
                                    ref.data(), &L) == 0);
    CHECK(std::size_t(L) == r.levels);
    std::size_t off = 0;
    for (const auto &c : r.classes) {
      CHECK(std::memcmp(c.data(), ref.data() + off, c.size() * sizeof(double)) == 0);
      off += c.size();
    }
    try {
      mgr::decompose_spatiotemporal(std::vector<mgr::TensorGrid<double>>{snaps[0]}, {0.0});
      CHECK(false);
    } catch (const mgr::ShapeError &e) {
      CHECK(e.code() == "ShapeError");
    }
  }
  // errors keep the reference's types and codes
  try {
    mgr::make_grid<double>({2, 2}, std::vector<double>(4));
    CHECK(false);
  } catch (const mgr::InvalidGrid &e) {
    CHECK(e.code() == "InvalidGrid");
  }
  {
    const auto g = mgr::make_grid<double>({9, 9}, std::vector<double>(81, 1.0));
    const auto r = mgr::decompose(g);
    try {
      mgr::recompose(r, r.levels + 1);
      CHECK(false);
    } catch (const mgr::InvalidLevel &e) {
      CHECK(e.code() == "InvalidLevel");
    }
    auto cut = r;
    cut.classes.resize(2);
    try {
      mgr::recompose(cut, 3);
      CHECK(false);
    } catch (const mgr::MissingClass &e) {
      CHECK(e.code() == "MissingClass");
    }
  }
  // embarrassing_decompose: result i == decompose(blocks[i])
  {
    std::vector<mgr::TensorGrid<double>> blocks;
    for (unsigned i = 0; i < 3; ++i) {
      std::vector<double> v(17 * 9);
      for (std::size_t k = 0; k < v.size(); ++k)
        v[k] = std::sin(0.1 * double(k + i));
      blocks.push_back(mgr::make_grid<double>({17, 9}, v));
    }
    const auto res = mgr::embarrassing_decompose(blocks, 2);
    for (std::size_t i = 0; i < blocks.size(); ++i) {
      const auto one = mgr::decompose(blocks[i]);
      CHECK(res[i].classes == one.classes);
    }
  }
  std::printf("shim ok\n");
  return 0;
}
