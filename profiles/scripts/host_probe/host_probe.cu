// Host-transfer probe for the pageable drop-in path (1025^3 f32 = 4.31 GB):
// pageable cudaMemcpy H2D/D2H, cudaHostRegister/Unregister cost, host memcpy
// bandwidth by thread count, pinned H2D/D2H.  nvcc -O2 -std=c++17 host_probe.cu
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      std::printf("%s: %s\n", #x, cudaGetErrorString(e_));                                \
      std::exit(1);                                                                        \
    }                                                                                      \
  } while (0)

static void pmemcpy(char *d, const char *s, size_t n, int T) {
  std::vector<std::thread> th;
  const size_t per = (n + T - 1) / T;
  for (int t = 0; t < T; ++t) {
    const size_t a = std::min(n, per * t), b = std::min(n, per * (t + 1));
    th.emplace_back([=] { std::memcpy(d + a, s + a, b - a); });
  }
  for (auto &x : th)
    x.join();
}

int main(int argc, char **argv) {
  const size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : size_t(1025) * 1025 * 1025 * 4;
  std::printf("{\"bytes\": %zu, \"hw_threads\": %u", n, std::thread::hardware_concurrency());
  char *d = nullptr;
  CK(cudaMalloc(&d, n));
  char *a = static_cast<char *>(std::malloc(n)), *b = static_cast<char *>(std::malloc(n));
  std::memset(a, 1, n);
  std::memset(b, 2, n);
  double t = now();
  CK(cudaMemcpy(d, a, n, cudaMemcpyHostToDevice));
  std::printf(", \"pageable_h2d_GBps\": %.2f", n / (now() - t) / 1e9);
  t = now();
  CK(cudaMemcpy(d, a, n, cudaMemcpyHostToDevice));
  std::printf(", \"pageable_h2d_GBps_2\": %.2f", n / (now() - t) / 1e9);
  t = now();
  CK(cudaMemcpy(b, d, n, cudaMemcpyDeviceToHost));
  std::printf(", \"pageable_d2h_GBps\": %.2f", n / (now() - t) / 1e9);
  t = now();
  CK(cudaHostRegister(a, n, cudaHostRegisterDefault));
  const double treg = now() - t;
  std::printf(", \"register_s\": %.4f", treg);
  t = now();
  CK(cudaMemcpy(d, a, n, cudaMemcpyHostToDevice));
  std::printf(", \"registered_h2d_GBps\": %.2f", n / (now() - t) / 1e9);
  t = now();
  CK(cudaHostUnregister(a));
  std::printf(", \"unregister_s\": %.4f", now() - t);
  // fresh (untouched) pages: register cost includes faulting them in
  char *c = static_cast<char *>(std::malloc(n));
  t = now();
  CK(cudaHostRegister(c, n, cudaHostRegisterDefault));
  std::printf(", \"register_untouched_s\": %.4f", now() - t);
  t = now();
  CK(cudaMemcpy(c, d, n, cudaMemcpyDeviceToHost));
  std::printf(", \"registered_d2h_GBps\": %.2f", n / (now() - t) / 1e9);
  CK(cudaHostUnregister(c));
  std::free(c);
  for (int T : {1, 2, 4, 8, 16, 32}) {
    t = now();
    pmemcpy(b, a, n, T);
    std::printf(", \"memcpy_T%d_GBps\": %.2f", T, n / (now() - t) / 1e9);
  }
  // a vector-like fresh allocation zero-filled (std::vector<float>(n))
  t = now();
  char *z = static_cast<char *>(std::calloc(n, 1));
  std::memset(z, 0, n);
  std::printf(", \"zero_fill_fresh_s\": %.4f", now() - t);
  std::free(z);
  char *p = nullptr;
  CK(cudaMallocHost(&p, n));
  std::memset(p, 0, n);
  t = now();
  CK(cudaMemcpy(d, p, n, cudaMemcpyHostToDevice));
  std::printf(", \"pinned_h2d_GBps\": %.2f", n / (now() - t) / 1e9);
  t = now();
  CK(cudaMemcpy(p, d, n, cudaMemcpyDeviceToHost));
  std::printf(", \"pinned_d2h_GBps\": %.2f", n / (now() - t) / 1e9);
  std::printf("}\n");
  return 0;
}
