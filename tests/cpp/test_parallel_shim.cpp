// C++ drop-in check of the parallel API (mgr/parallel.hpp): code written
// against the reference's cooperative_decompose / grouped_decompose /
// make_partitions, compiled against include/mgr_b200/parallel.hpp, classes
// compared bit-for-bit with the reference library's serial decompose
// (test_parallel.cpp:88-240).  Build + run: tests/test_cpp_shim.py.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <set>

#include "mgr_b200/parallel.hpp"

extern "C" int mgrref_decompose_f64(int, const uint64_t *, const double *, int, const double *,
                                    double *, int *);

#define CHECK(c)                                                               \
  do {                                                                         \
    if (!(c)) {                                                                \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);\
      std::exit(1);                                                            \
    }                                                                          \
  } while (0)

static mgr::TensorGrid<double> random_grid(const mgr::Shape &shape, unsigned seed) {
  std::mt19937 gen(seed);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  std::vector<double> v(mgr::num_elements(shape));
  for (auto &x : v)
    x = U(gen);
  return mgr::make_grid<double>(shape, v);
}

static void equals_reference_serial(const mgr::TensorGrid<double> &g,
                                    const mgr::RefactoredData<double> &r, int cap = 0) {
  std::vector<uint64_t> sh(g.shape.begin(), g.shape.end());
  std::vector<double> cf;
  for (const auto &c : g.coords)
    cf.insert(cf.end(), c.begin(), c.end());
  std::vector<double> ref(g.values.size());
  int L = 0;
  CHECK(mgrref_decompose_f64(int(sh.size()), sh.data(), cf.data(), cap, g.values.data(),
                             ref.data(), &L) == 0);
  CHECK(std::size_t(L) == r.levels);
  std::size_t off = 0;
  for (const auto &c : r.classes) {
    CHECK(std::memcmp(c.data(), ref.data() + off, c.size() * sizeof(double)) == 0);
    off += c.size();
  }
  CHECK(off == ref.size());
}

int main() {
  using namespace mgr;
  // partitions (test_parallel.cpp:32-86)
  {
    const auto p = make_partitions(Shape{9, 9, 9}, 3, PartitionScheme::block);
    CHECK(p.size() == 3 && p[1].lo[2] == 3 && p[1].hi[2] == 6 && p[2].worker == 2);
    const auto s = make_partitions(Shape{9, 9}, 3, PartitionScheme::shifted_round_robin);
    CHECK(s.size() == 9);
    for (const auto &q : s)
      CHECK(q.worker == int((q.block_coord[0] + q.block_coord[1]) % 3));
    try {
      make_partitions(Shape{9, 9}, 10, PartitionScheme::block);
      CHECK(false);
    } catch (const TooManyWorkers &e) {
      CHECK(e.code() == "TooManyWorkers");
    }
    try {
      make_partitions(Shape{9}, 2, PartitionScheme::shifted_round_robin);
      CHECK(false);
    } catch (const ShapeError &) {
    }
  }
  // cooperative == serial for every configuration (test_parallel.cpp:95-108)
  {
    const auto g = random_grid(Shape{17, 17, 17}, 61);
    for (PartitionScheme sc : {PartitionScheme::block, PartitionScheme::shifted_round_robin})
      for (int w : {1, 2, 3, 4}) {
        CoopOptions o;
        o.scheme = sc;
        CommReport rep;
        o.report = &rep;
        const auto r = cooperative_decompose(g, w, o);
        equals_reference_serial(g, r);
        CHECK(rep.workers == w);
      }
    const auto big = random_grid(Shape{33, 17, 65}, 7);
    equals_reference_serial(big, cooperative_decompose(big, 5));
  }
  // non-dyadic extents and level caps (test_parallel.cpp:110-123)
  {
    const auto g = random_grid(Shape{12, 10, 9}, 62);
    CoopOptions o;
    o.levels = 2;
    o.scheme = PartitionScheme::shifted_round_robin;
    equals_reference_serial(g, cooperative_decompose(g, 3, o), 2);
  }
  // constant fields: zero classes under any worker count
  {
    const auto g = make_grid<double>(Shape{9, 9, 9}, std::vector<double>(729, 1.5));
    for (int w : {2, 4}) {
      const auto r = cooperative_decompose(g, w);
      for (std::size_t l = 1; l <= r.levels; ++l)
        for (double c : r.classes[l])
          CHECK(c == 0.0);
    }
  }
  // fault injection surfaces as WorkerFailure (test_parallel.cpp:190-205)
  {
    const auto g = random_grid(Shape{17, 17, 17}, 63);
    CoopOptions o;
    o.fault_injector = [](int w, const std::string &phase, std::size_t) {
      if (w == 1 && phase == "solve")
        throw std::runtime_error("injected");
    };
    try {
      cooperative_decompose(g, 3, o);
      CHECK(false);
    } catch (const WorkerFailure &e) {
      CHECK(e.code() == "WorkerFailure");
    }
  }
  // grouped mode (test_parallel.cpp:225-240)
  {
    std::vector<TensorGrid<double>> blocks;
    for (unsigned i = 0; i < 4; ++i)
      blocks.push_back(random_grid(Shape{9, 9, 9}, 80 + i));
    const auto res = grouped_decompose(blocks, 2, 2);
    CHECK(res.size() == 4);
    for (std::size_t i = 0; i < blocks.size(); ++i)
      equals_reference_serial(blocks[i], res[i]);
  }
  std::printf("parallel shim ok\n");
  return 0;
}
