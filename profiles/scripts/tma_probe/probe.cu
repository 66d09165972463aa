// TMA 1-D tiled-map probe: which (dim, box, coordinate) combinations load.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "tma.cuh"
using namespace mgrg;
__global__ void k(const __grid_constant__ CUtensorMap m, int c, double *out) {
  __shared__ __align__(128) double buf[32];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  fence_barrier_init();
  __syncwarp();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, 256);
    tma_load_1d(buf, &m, c, &bar);
  }
  mbar_wait(&bar, 0);
  out[threadIdx.x] = buf[threadIdx.x];
}
int main(int argc, char **argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  void *f = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)f;
  double *d, *o; cudaMalloc(&d, 1 << 20); cudaMalloc(&o, 256);
  std::vector<double> h(1 << 17); for (size_t i = 0; i < h.size(); ++i) h[i] = double(i);
  cudaMemcpy(d, h.data(), 1 << 20, cudaMemcpyHostToDevice);
  struct C { unsigned long long dim; int c; bool gs; } cs[] = {
    {4096, 0, true}, {4096, 5, true}, {4096, -3, true}, {4096, 4090, true}, {15, 0, true},
    {31, 0, true}, {32, 0, true}, {4096, 0, false}, {15, 0, false}, {4096, 2, true},
    {4096, 1, true}, {4096, -2, true}, {4096, 4094, true}};
  int idx = -1;
  for (auto cc : cs) {
    if (only >= 0 && ++idx != only) continue;
    CUtensorMap m; cuuint64_t gd[1] = {cc.dim}, gsd[1] = {cc.dim * 8}; cuuint32_t bd[1] = {32}, es[1] = {1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, d, gd, cc.gs ? gsd : nullptr, bd, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaMemset(o, 0xff, 256);
    k<<<1, 32>>>(m, cc.c, o);
    cudaError_t e = cudaDeviceSynchronize();
    double r8[32]; cudaMemcpy(r8, o, 256, cudaMemcpyDeviceToHost);
    printf("dim %llu c %d gs %d: encode %d launch %s  v0 %g v1 %g v31 %g\n", cc.dim, cc.c, cc.gs, int(r),
           cudaGetErrorString(e), r8[0], r8[1], r8[31]);
    if (e != cudaSuccess) return 1;
  }
  // L2 promotion variants
  for (auto l2 : {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B}) {
    CUtensorMap m; cuuint64_t gd[1] = {4096}, gsd[1] = {4096 * 8}; cuuint32_t bd[1] = {32}, es[1] = {1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, d, gd, gsd, bd, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k<<<1, 32>>>(m, 3, o);
    cudaError_t e = cudaDeviceSynchronize();
    printf("l2 %d: encode %d launch %s\n", int(l2), int(r), cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
