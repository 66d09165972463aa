// End-to-end timing of the C++ source drop-in as a reference caller uses it
// (include/mgr_b200/refactor.hpp): pageable std::vector input, per-class
// std::vector output, mgr::decompose then mgr::recompose with every class
// (refactor.hpp:462-496 call shapes), wall-clocked per step on the host.
//   bench_dropin <n> <steps> <warmup> <fast 0|1>  ->  one JSON line
// Built and run by bench.py (the "dropin_e2e" key); not a test.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#include "mgr_b200/refactor.hpp"

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

int main(int argc, char **argv) {
  const std::size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1025;
  const int steps = argc > 2 ? std::atoi(argv[2]) : 3;
  const int warmup = argc > 3 ? std::atoi(argv[3]) : 1;
  const bool fast = argc > 4 && std::atoi(argv[4]) != 0;
  // bench.py's smooth field family (acceptance.cpp:383-393 shape), block 0
  std::vector<float> v(n * n * n);
  {
    std::vector<double> e1(n), e2(n), s(n);
    const double c1 = 0.4, c2 = 0.65;
    for (std::size_t i = 0; i < n; ++i) {
      const double x = double(i) / double(n - 1) / 2.0;
      e1[i] = std::exp(-30 * (x - c1) * (x - c1));
      e2[i] = std::exp(-25 * (x - c2) * (x - c2));
      s[i] = std::sin(2 * M_PI * x);
    }
    const unsigned T = std::max(1u, std::thread::hardware_concurrency());
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        for (std::size_t z = t; z < n; z += T)
          for (std::size_t y = 0; y < n; ++y)
            for (std::size_t x = 0; x < n; ++x)
              v[(z * n + y) * n + x] = float(e1[x] * e1[y] * e1[z] +
                                             0.6 * e2[x] * e2[y] * e2[z] +
                                             0.2 * s[x] * s[y] * s[z]);
      });
    for (auto &x : th)
      x.join();
  }
  mgr::TensorGrid<float> grid = mgr::make_grid<float>({n, n, n}, std::move(v));
  mgr::RefactorOptions opt;
  opt.fast = fast;
  double tdec = 0, trec = 0, err = 0;
  for (int it = 0; it < warmup + steps; ++it) {
    const double t0 = now();
    mgr::RefactoredData<float> r = mgr::decompose(grid, opt);
    const double t1 = now();
    mgr::TensorGrid<float> back = mgr::recompose(r, r.levels, opt);
    const double t2 = now();
    if (it >= warmup) {
      tdec += t1 - t0;
      trec += t2 - t1;
    }
    if (it == warmup + steps - 1)
      for (std::size_t i = 0; i < back.values.size(); i += 997)
        err = std::max(err, double(std::fabs(back.values[i] - grid.values[i])));
  }
  // the same two calls through the C ABI into caller buffers that already
  // exist (pageable, touched): transfers + device work without the output
  // allocation the reference API's by-value results impose
  double t_reuse = 0;
  {
    mgr::RefactoredData<float> r = mgr::decompose(grid, opt);
    mgrg_plan *p = mgr::b200_detail::plan_for<float>(grid.shape, grid.coords, std::nullopt, 0, fast);
    std::vector<void *> dst;
    std::vector<const void *> src;
    for (auto &c : r.classes) {
      dst.push_back(c.data());
      src.push_back(c.data());
    }
    std::vector<float> back(grid.values.size());
    for (int it = 0; it < 1 + steps; ++it) {
      const double t0 = now();
      mgr::b200_detail::check(mgrg_decompose_host_classes(p, grid.values.data(), dst.data()));
      mgr::b200_detail::check(
          mgrg_recompose_host_classes(p, src.data(), int32_t(r.levels), back.data()));
      if (it > 0)
        t_reuse += now() - t0;
    }
  }
  // the output-allocation floor: the reference API returns the classes and
  // the field in fresh std::vectors (value-initialised: page faults + zero fill)
  double t_plain = 0, t_pref = 0;
  {
    const double t0 = now();
    { std::vector<float> a(n * n * n); }
    const double t1 = now();
    { std::vector<float> b = mgr::b200_detail::make_output_vector<float>(n * n * n); }
    const double t2 = now();
    t_plain = t1 - t0;
    t_pref = t2 - t1;
  }
  const double bytes = double(n) * n * n * sizeof(float);
  std::printf("{\"n\": %zu, \"fast\": %d, \"steps\": %d, \"decompose_ms\": %.2f, "
              "\"recompose_ms\": %.2f, \"ms_per_step\": %.2f, \"GBps\": %.3f, "
              "\"decompose_GBps\": %.3f, \"recompose_GBps\": %.3f, \"roundtrip_max_err\": %.3g, "
              "\"alloc_vector_ms\": %.1f, \"alloc_prefaulted_ms\": %.1f, "
              "\"capi_reused_buffers_ms_per_step\": %.2f}\n",
              n, int(fast), steps, 1e3 * tdec / steps, 1e3 * trec / steps,
              1e3 * (tdec + trec) / steps, 2 * bytes * steps / (tdec + trec) / 1e9,
              bytes * steps / tdec / 1e9, bytes * steps / trec / 1e9, err, 1e3 * t_plain,
              1e3 * t_pref, 1e3 * t_reuse / steps);
  return 0;
}
