#include <chrono>
#include <cstdio>
#include <vector>
#include "mgr_b200/refactor.hpp"
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
  const size_t n = size_t(1025) * 1025 * 1025;
  for (int rep = 0; rep < 2; ++rep) {
    double t0 = now();
    std::vector<float> v;
    v.reserve(n);
    double t1 = now();
    mgr::b200_detail::prefault(v.data(), n * sizeof(float));
    double t2 = now();
    v.resize(n);
    double t3 = now();
    std::vector<float> w(n);
    double t4 = now();
    { std::vector<float> x; x.reserve(n); x.resize(n); }
    double t5 = now();
    std::printf("{\"reserve_ms\": %.1f, \"populate_ms\": %.1f, \"resize_ms\": %.1f, \"plain_ms\": %.1f, \"reserve_resize_ms\": %.1f}\n",
                1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t4 - t3), 1e3 * (t5 - t4));
  }
}
