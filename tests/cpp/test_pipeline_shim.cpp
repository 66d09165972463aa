// C++ drop-in check for the pipeline API: code written against the
// reference's mgr/pipeline.hpp (crc32, write_refactored, read_refactored,
// read_refactored_header, compress, decompress) compiled against
// include/mgr_b200/pipeline.hpp; files and compressed containers compared
// byte-for-byte with the reference library's (oracle/_ref C harness -- test
// infrastructure).  Build + run: tests/test_cpp_shim.py.  Prints "pipeline ok".
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <random>

#include "mgr_b200/pipeline.hpp"

extern "C" {
int64_t mgrref_write_refactored_f64(int, const uint64_t *, const double *, int, const double *,
                                    const char *);
int64_t mgrref_compress_f64(int, const uint64_t *, const double *, const double *, double, int,
                            uint8_t *, uint64_t, double *, double *);
int64_t mgrref_decompress(const uint8_t *, uint64_t, void *, uint64_t);
uint32_t mgrref_crc32(const uint8_t *, uint64_t);
}

#define CHECK(c)                                                               \
  do {                                                                         \
    if (!(c)) {                                                                \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);\
      std::exit(1);                                                            \
    }                                                                          \
  } while (0)

static std::vector<uint8_t> slurp(const std::string &p) {
  std::ifstream in(p, std::ios::binary);
  return {std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()};
}

int main(int argc, char **argv) {
  const std::string dir = argc > 1 ? argv[1] : "/tmp";
  std::mt19937 gen(7);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  const mgr::Shape shape{17, 9, 5};
  std::vector<double> v(mgr::num_elements(shape));
  for (auto &x : v)
    x = U(gen);
  const auto g = mgr::make_grid<double>(shape, v);
  const auto r = mgr::decompose(g);
  // container: write, compare with the reference writer, read back
  const std::string ours = dir + "/shim_ours.mgrf", ref = dir + "/shim_ref.mgrf";
  const auto n = mgr::write_refactored(r, ours);
  std::vector<double> flat;
  for (const auto &c : r.classes)
    flat.insert(flat.end(), c.begin(), c.end());
  std::vector<uint64_t> sh(shape.begin(), shape.end());
  std::vector<double> cf;
  for (const auto &c : g.coords)
    cf.insert(cf.end(), c.begin(), c.end());
  CHECK(mgrref_write_refactored_f64(3, sh.data(), cf.data(), int(r.levels), flat.data(),
                                    ref.c_str()) == int64_t(n));
  CHECK(slurp(ours) == slurp(ref));
  const auto h = mgr::read_refactored_header(ours);
  CHECK(h.levels == r.levels && h.shape == shape && h.dtype == mgr::DType::f64);
  const auto rr = mgr::read_refactored(ours, 1);
  CHECK(rr.classes_loaded == 1);
  const auto &rd = std::get<mgr::RefactoredData<double>>(rr.data);
  CHECK(rd.classes.size() == 2 && rd.classes[1] == r.classes[1]);
  const auto bytes = slurp(ours);
  CHECK(mgr::crc32(bytes) == mgrref_crc32(bytes.data(), bytes.size()));
  try {
    mgr::read_refactored(ours, r.levels + 1);
    CHECK(false);
  } catch (const mgr::MissingClass &e) {
    CHECK(std::string(e.code()) == "MissingClass");
  }
  // compression: identical containers, identical decompressed values
  for (const auto *codec : {&mgr::store_codec(), &mgr::zlib_codec()}) {
    const auto c = mgr::compress(g, 1e-3, *codec);
    std::vector<uint8_t> rb(1 << 20);
    double bin = 0, meas = 0;
    const int64_t m = mgrref_compress_f64(3, sh.data(), cf.data(), v.data(), 1e-3, codec->id(),
                                          rb.data(), rb.size(), &bin, &meas);
    CHECK(m > 0);
    rb.resize(std::size_t(m));
    CHECK(c.bytes == rb);
    CHECK(c.report.bin_width == bin && c.report.measured_max_abs_error == meas);
    const auto d = mgr::decompress(c.bytes);
    const auto &dg = std::get<mgr::TensorGrid<double>>(d.grid);
    std::vector<double> refv(v.size());
    CHECK(mgrref_decompress(rb.data(), rb.size(), refv.data(), refv.size()) == 0);
    CHECK(dg.values == refv);
  }
  try {
    mgr::compress(g, 0.0);
    CHECK(false);
  } catch (const mgr::InvalidBound &) {
  }
  std::printf("pipeline ok\n");
  return 0;
}
