// Cost of materialising a fresh 4.3 GB std::vector<float> the way the drop-in
// does (reserve, fault the pages in, value-initialise) by fault strategy.
#include <sys/mman.h>

#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>
static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
#ifndef MADV_POPULATE_WRITE
#define MADV_POPULATE_WRITE 23
#endif
static double populate(void *p, size_t bytes, unsigned T, bool huge) {
  const double t0 = now();
  const size_t pg = 4096;
  const uintptr_t a = (reinterpret_cast<uintptr_t>(p) + pg - 1) & ~(pg - 1);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes) & ~(pg - 1);
  if (huge)
    madvise(reinterpret_cast<void *>(a), e - a, MADV_HUGEPAGE);
  const size_t per = ((e - a) / T + (2u << 20) - 1) & ~size_t((2u << 20) - 1);
  std::vector<std::thread> th;
  for (unsigned t = 0; t < T; ++t) {
    const uintptr_t s0 = a + t * per, s1 = std::min<uintptr_t>(e, s0 + per);
    if (s1 > s0)
      th.emplace_back([=] { madvise(reinterpret_cast<void *>(s0), s1 - s0, MADV_POPULATE_WRITE); });
  }
  for (auto &x : th)
    x.join();
  return now() - t0;
}
int main() {
  const size_t n = size_t(1025) * 1025 * 1025;
  for (bool huge : {false, true})
    for (unsigned T : {1u, 4u, 16u}) {
      std::vector<float> v;
      v.reserve(n);
      const double tp = populate(v.data(), n * sizeof(float), T, huge);
      const double t0 = now();
      v.resize(n);
      const double tr = now() - t0;
      std::printf("{\"huge\": %d, \"threads\": %u, \"populate_ms\": %.1f, \"resize_ms\": %.1f}\n", int(huge), T,
                  1e3 * tp, 1e3 * tr);
    }
  FILE *f = std::fopen("/sys/kernel/mm/transparent_hugepage/enabled", "r");
  char buf[256] = {0};
  if (f) { std::fgets(buf, sizeof buf, f); std::fclose(f); }
  std::printf("thp: %s", buf);
  f = std::fopen("/sys/kernel/mm/transparent_hugepage/defrag", "r");
  if (f) { std::fgets(buf, sizeof buf, f); std::fclose(f); }
  std::printf("defrag: %s", buf);
}
