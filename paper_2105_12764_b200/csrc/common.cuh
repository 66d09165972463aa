// common.cuh -- device helpers shared by the refactoring kernels.
//
// Arithmetic goes through the _rn intrinsics so ptxas never contracts a
// multiply into an FMA: every kernel evaluates the reference expression
// (/root/reference/proj/include/mgr/kernels.hpp) in the same order with the
// same roundings, which makes the device path bit-identical to the
// reference CPU path (built without -march, i.e. without FMA).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace mgrg {

template <typename R> __device__ __forceinline__ R mul(R a, R b);
template <> __device__ __forceinline__ float mul<float>(float a, float b) {
  return __fmul_rn(a, b);
}
template <> __device__ __forceinline__ double mul<double>(double a, double b) {
  return __dmul_rn(a, b);
}
template <typename R> __device__ __forceinline__ R add(R a, R b);
template <> __device__ __forceinline__ float add<float>(float a, float b) {
  return __fadd_rn(a, b);
}
template <> __device__ __forceinline__ double add<double>(double a, double b) {
  return __dadd_rn(a, b);
}
template <typename R> __device__ __forceinline__ R sub(R a, R b);
template <> __device__ __forceinline__ float sub<float>(float a, float b) {
  return __fsub_rn(a, b);
}
template <> __device__ __forceinline__ double sub<double>(double a, double b) {
  return __dsub_rn(a, b);
}

// a + t*(b - a)  (kernels.hpp:219)
template <typename R> __device__ __forceinline__ R lerp(R a, R b, R t) {
  return add(a, mul(t, sub(b, a)));
}

// Position helpers (grid.hpp:74-85).  They are also correct for dimensions
// that never refine (extent 1 or 2): every position is coarse there and
// coarse_rank/coarse_pos are the identity.
__device__ __forceinline__ bool is_coarse(uint32_t p, uint32_t n) {
  return (p & 1u) == 0 || p == n - 1;
}
__device__ __forceinline__ uint32_t coarse_rank(uint32_t p) {
  return (p & 1u) == 0 ? p >> 1 : (p >> 1) + 1;
}
__device__ __forceinline__ uint32_t fine_rank(uint32_t p) { return (p - 1) >> 1; }
__device__ __forceinline__ uint32_t coarse_pos(uint32_t k, uint32_t n) {
  return 2 * k < n - 1 ? 2 * k : n - 1;
}

// Merged mass-trans output for kept index i of one fiber
// (masstrans_window, kernels.hpp:159-178):
//   v = mv(q) [+ r[q-2]*mv(q-1)] [+ (1-r[q])*mv(q+1)],  q = coarse_pos(i)
//   mv(j) = h[j-1]*in(j-1) + 2(h[j-1]+h[j])*in(j) + h[j]*in(j+1)
// `in(j)` takes the fiber position; `h`/`r` are the level spacings/ratios
// of this dimension in the working precision.
template <typename R, typename In>
__device__ __forceinline__ R masstrans_at(In &&in, uint32_t q, uint32_t n,
                                          const R *__restrict__ h,
                                          const R *__restrict__ r) {
  auto mv = [&](uint32_t j) -> R {
    if (j == 0) {
      const R h0 = __ldg(h);
      return add(mul(mul(R(2), h0), in(0)), mul(h0, in(1)));
    }
    if (j == n - 1) {
      const R hl = __ldg(h + n - 2);
      return add(mul(hl, in(n - 2)), mul(mul(R(2), hl), in(n - 1)));
    }
    const R ha = __ldg(h + j - 1), hb = __ldg(h + j);
    return add(add(mul(ha, in(j - 1)), mul(mul(R(2), add(ha, hb)), in(j))),
               mul(hb, in(j + 1)));
  };
  R v = mv(q);
  if (q >= 1 && !is_coarse(q - 1, n))
    v = add(v, mul(__ldg(r + q - 2), mv(q - 1)));
  if (q + 1 < n && !is_coarse(q + 1, n))
    v = add(v, mul(sub(R(1), __ldg(r + q)), mv(q + 1)));
  return v;
}

// cp.async helpers (LDGSTS): element-granular async global->shared copies;
// the level arrays have odd row pitches (e.g. 1025 elements), which rules
// out 16-byte TMA tensor maps, so the staging uses 4/8-byte LDGSTS.
template <typename R>
__device__ __forceinline__ void cp_async(R *smem, const R *gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  if constexpr (sizeof(R) == 4)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
// 16-byte LDGSTS (both addresses 16-byte aligned), L2-only caching.
template <typename R>
__device__ __forceinline__ void cp_async16(R *smem, const R *gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::);
}
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Programmatic dependent launch: kernels of the level loop are launched
// with programmatic stream serialization, so a kernel's CTAs are scheduled
// while its predecessor drains; every such kernel waits here (first
// statement) until the predecessor's writes are visible.  A no-op for
// ordinary launches.
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

} // namespace mgrg
