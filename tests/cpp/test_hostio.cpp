// CPU unit test of the host side of the host-buffer C ABI (csrc/hostio.cuh):
// the HostView piece split across per-class buffers and the parallel copy
// pool.  No device calls.  Built and run by tests/test_capi.py.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <random>
#include <vector>

#include "../../paper_2105_12764_b200/csrc/hostio.cuh"

#define CHECK(c)                                                                            \
  do {                                                                                      \
    if (!(c)) {                                                                             \
      std::fprintf(stderr, "%s:%d CHECK failed: %s\n", __FILE__, __LINE__, #c);            \
      std::exit(1);                                                                         \
    }                                                                                       \
  } while (0)

int main() {
  using mgrg::HostView;
  // classes of 1, 7, 56, 448 elements (a 3-level 1-D-like layout) + an empty class
  const std::vector<uint64_t> sizes = {1, 7, 0, 56, 448};
  std::vector<uint64_t> off(sizes.size() + 1, 0);
  for (size_t l = 0; l < sizes.size(); ++l)
    off[l + 1] = off[l] + sizes[l];
  const uint64_t N = off.back();
  std::vector<std::vector<float>> cls(sizes.size());
  for (size_t l = 0; l < sizes.size(); ++l)
    cls[l].assign(sizes[l], 0.f);
  HostView v;
  v.es = sizeof(float);
  for (size_t l = 0; l < sizes.size(); ++l) {
    v.seg.push_back(reinterpret_cast<char *>(cls[l].data()));
    v.off.push_back(off[l]);
  }
  v.off.push_back(N);
  // every [o, o + n) range: the pieces tile it exactly, in order, and land
  // in the right class at the right place
  std::mt19937 rng(7);
  for (int trial = 0; trial < 2000; ++trial) {
    const uint64_t o = rng() % (N + 1), n = rng() % (N - o + 1);
    uint64_t covered = 0;
    v.pieces(o, n, [&](char *h, uint64_t at, uint64_t len) {
      CHECK(at == covered);
      CHECK(len > 0);
      const uint64_t g = o + at; // flat element index of the piece start
      size_t l = 0;
      while (!(g >= off[l] && g < off[l + 1]))
        ++l;
      CHECK(g + len <= off[l + 1]);
      CHECK(h == reinterpret_cast<char *>(cls[l].data()) + (g - off[l]) * sizeof(float));
      covered += len;
    });
    CHECK(covered == n);
  }
  // flat view: one piece
  std::vector<float> flat(N);
  HostView f;
  f.es = sizeof(float);
  f.flat = reinterpret_cast<char *>(flat.data());
  int np = 0;
  f.pieces(3, 100, [&](char *h, uint64_t at, uint64_t len) {
    CHECK(h == f.flat + 3 * sizeof(float) && at == 0 && len == 100);
    ++np;
  });
  CHECK(np == 1);
  // parallel copy pool: sizes around the split thresholds, odd offsets
  for (size_t n : {size_t(0), size_t(1), size_t(4097), size_t(1) << 20, (size_t(3) << 20) + 13,
                   size_t(67) << 20}) {
    std::vector<unsigned char> src(n + 3), dst(n + 3, 0xAB);
    for (size_t i = 0; i < src.size(); ++i)
      src[i] = static_cast<unsigned char>(i * 131 + 7);
    mgrg::CopyPool::get().copy(dst.data() + 1, src.data() + 2, n);
    CHECK(dst[0] == 0xAB && dst[n + 1] == 0xAB);
    CHECK(std::memcmp(dst.data() + 1, src.data() + 2, n) == 0);
  }
  std::printf("hostio ok\n");
  return 0;
}
