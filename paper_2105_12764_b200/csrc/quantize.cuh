// quantize.cuh -- device kernels of the compression pipeline (SURVEY.md §8(f)
// row 2; reference src/pipeline.cpp:381-440, include/mgr/pipeline.hpp:149-198):
//   quantize_class  q = llround(double(v) / bin), dequantized Real(double(q) * bin)
//   max |a - b| in double (the measured round-trip error of compress)
//   zigzag + base-128 varint encode (per-element byte lengths, exclusive scan,
//   scatter) and decode (terminator scan, per-element decode), with the
//   reference decoder's error semantics (truncated / overflow / trailing).
// All element-parallel, HBM-bound; exact integer/IEEE arithmetic, so the
// results are bit-identical to the reference's sequential loops.
#pragma once

#include <cstdint>

namespace mgrg {

template <typename R>
__global__ void quantize_kernel(const R *__restrict__ v, uint64_t n, double bin,
                                int64_t *__restrict__ q, R *__restrict__ deq) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const long long k = llround(double(v[i]) / bin); // pipeline.cpp:387-388
    if (q)
      q[i] = k;
    if (deq)
      deq[i] = R(double(k) * bin); // pipeline.hpp:168
  }
}

template <typename R>
__global__ void dequantize_kernel(const int64_t *__restrict__ q, uint64_t n, double bin,
                                  R *__restrict__ out) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = R(double(q[i]) * bin); // pipeline.cpp:534
}

// max |double(a) - double(b)| (NaN differences ignored, as std::max keeps
// the running value, pipeline.hpp:170-173); non-negative doubles order like
// their bit patterns, so the block maxima meet in one atomicMax.
template <typename R>
__global__ void maxabs_kernel(const R *__restrict__ a, const R *__restrict__ b, uint64_t n,
                              unsigned long long *__restrict__ out) {
  double m = 0.0;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    m = fmax(m, fabs(double(a[i]) - double(b[i])));
  for (int o = 16; o; o >>= 1)
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double wm[32];
  if ((threadIdx.x & 31) == 0)
    wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < int(blockDim.x >> 5); ++w)
      m = fmax(m, wm[w]);
    atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(m)));
  }
}

__device__ __forceinline__ uint64_t zz(int64_t v) {
  return (static_cast<uint64_t>(v) << 1) ^ static_cast<uint64_t>(v >> 63); // :397-399
}
__device__ __forceinline__ uint32_t varint_len(uint64_t u) {
  const int bits = 64 - __clzll(u | 1);
  return uint32_t((bits + 6) / 7);
}

__global__ void zz_len_kernel(const int64_t *__restrict__ q, uint64_t n,
                              uint64_t *__restrict__ len) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    len[i] = varint_len(zz(q[i]));
}

// off = exclusive prefix sum of the lengths (n + 1 entries, off[n] = total)
__global__ void zz_write_kernel(const int64_t *__restrict__ q, uint64_t n,
                                const uint64_t *__restrict__ off, uint8_t *__restrict__ out) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t u = zz(q[i]);
    uint8_t *p = out + off[i];
    while (u >= 0x80) { // pipeline.cpp:400-404
      *p++ = uint8_t(u) | 0x80;
      u >>= 7;
    }
    *p = uint8_t(u);
  }
}

// term[i] = 1 when byte i ends an element (high bit clear)
__global__ void zz_term_kernel(const uint8_t *__restrict__ b, uint64_t nb,
                               uint64_t *__restrict__ term) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nb;
       i += uint64_t(gridDim.x) * blockDim.x)
    term[i] = (b[i] & 0x80) ? 0 : 1;
}

// rank = exclusive scan of term (nb + 1 entries): element e ends at the byte
// i with term[i] && rank[i] == e.  Decodes elements e < count whose end lies
// in the stream; records the first element longer than 10 bytes (the
// reference's "varint overflow", pipeline.cpp:425-426) in *bad.
__global__ void zz_decode_kernel(const uint8_t *__restrict__ b, uint64_t nb,
                                 const uint64_t *__restrict__ rank, uint64_t count,
                                 int64_t *__restrict__ q, unsigned long long *__restrict__ bad) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nb;
       i += uint64_t(gridDim.x) * blockDim.x) {
    if (b[i] & 0x80)
      continue;
    const uint64_t e = rank[i];
    if (e >= count)
      continue;
    // start: one past the previous terminator (elements are at most 10
    // bytes long unless corrupt)
    uint64_t s = i;
    int len = 1;
    while (s > 0 && (b[s - 1] & 0x80)) {
      --s;
      if (++len > 10)
        break;
    }
    if (len > 10) { // the 10th byte continues: the reference overflows
      atomicMin(bad, static_cast<unsigned long long>(e));
      continue;
    }
    uint64_t u = 0;
    int shift = 0;
    for (uint64_t k = s; k <= i; ++k, shift += 7)
      u |= uint64_t(b[k] & 0x7F) << shift;
    q[e] = static_cast<int64_t>(u >> 1) ^ -static_cast<int64_t>(u & 1); // :431-432
  }
}

} // namespace mgrg
