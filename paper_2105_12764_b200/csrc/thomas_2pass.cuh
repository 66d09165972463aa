// thomas_2pass.cuh -- FAST-policy Thomas solve of LONG fibers (more
// positions than one CTA holds: the long 2-D levels of 8193^2, 4097^2, ...)
// as two streaming passes over the lattice with a tiny carry solve between.
//
// The level-(l-1) mass matrix along a dimension is the same for every fiber
// (TridiagonalOperator::build, kernels.hpp:98-136), so with the sweeps of
// thomas_fiber (kernels.hpp:143-151) written as
//   forward : v_i = f_i + fwd_i * v_{i-1}
//   backward: x_i = ip_i * v_i + g_i * x_{i+1},   g_i = -ip_i * h_i
// a chunk [a, b) of a fiber (kTpC positions) depends on the rest of the fiber
// only through two scalars: c = v_{a-1} (forward carry-in) and d = x_b
// (backward carry-in).  With vl / xl the chunk solved from zero carries,
//   v_{b-1} = vl_{b-1} + PF * c                       PF = prod_{a..b-1} fwd
//   x_a     = xl_a     + Q  * c + PB * d              PB = prod_{a..b-1} g,
// Q = x_a of the backward sweep over v = (prod_{a..i} fwd)_i -- all three
// fiber-independent (host table).  So
//   pass 1 (tp_pass1_kernel): one read of f; per (chunk, fiber) the pair
//          E = vl_{b-1}, S = xl_a;
//   carry  (tp_carry_kernel): per fiber, c_{k+1} = PF_k c_k + E_k upward and
//          d_{k-1} = PB_k d_k + (S_k + Q_k c_k) downward, as affine-map warp
//          scans over 32 chunks at a time (in place: E -> c, S -> d);
//   pass 2 (tp_pass2_kernel): one read + one write of f; each chunk re-runs
//          the plain sequential sweeps from its exact carries (fused apply /
//          unapply epilogue on the last solve of a level).
// 3 streaming touches of the lattice instead of 2, but every pass is a
// simple stream (no fiber-sized on-chip state, no cluster barriers): 8193^2
// f64 level 13, y + apply 150 -> 112 us (pass 2 alone at 6.4 TB/s).
// Only the association of the recurrences changes: FAST tolerance, not
// bit-identity (the exact policy keeps the sequential kernels).
//
// Strided fibers only (same numbering as the other Thomas kernels): DIM 1
// fiber F = x + m0*z, positions m0 apart; DIM 2 fiber F = x + m0*y,
// positions m0*m1 apart.  Lane = fiber, so every position row of a warp is
// 32 consecutive fibers (coalesced).  Contiguous (x) fibers stay on the
// cluster kernel: a DIM-0 variant of these passes (chunks transposed through
// shared memory) measured slower there (profiles/r2/tuning/README.md).
#pragma once

#include "common.cuh"
#include "level.cuh"

namespace mgrg {

#ifndef TP_C
#define TP_C 16
#endif
#ifndef TP_MINB1
#define TP_MINB1 3 // CTAs per SM of pass 1
#endif
#ifndef TP_MINB2
#define TP_MINB2 2 // pass 2 (+ the epilogue bases: no spills at 2)
#endif
constexpr int kTpC = TP_C;    // positions per chunk (16: 3 CTAs per SM, loads of the
                              // next CTA overlap this one's sweeps; 32: one CTA per SM)
constexpr int kTpWarps = 8;   // fiber groups (warps) per CTA, all on the same chunk
constexpr int kTpMaxK = 512;  // chunks per fiber handled (carry scan registers)

// Host table: per position {fwd, ip, g, 0}, then per chunk {PF, Q, PB, 0}.
template <typename R> struct ThomasTP {
  const R *q;  // [4 m]
  const R *ck; // [4 K]
  uint32_t m, K;
  R *scratch; // host side: the plan's E / S scratch (2 * fibers * K elements)
};

template <int DIM>
__device__ __forceinline__ uint64_t tp_fiber_base(uint64_t F, uint32_t m0, uint32_t m1) {
  static_assert(DIM == 1 || DIM == 2, "strided fibers only");
  return DIM == 1 ? (F % m0) + uint64_t(m0) * m1 * (F / m0) : F;
}
template <int DIM> __device__ __forceinline__ uint64_t tp_stride(uint32_t m0, uint32_t m1) {
  return DIM == 1 ? uint64_t(m0) : uint64_t(m0) * m1;
}

// CTA = 8 groups of 32 adjacent fibers on one chunk (blockIdx.y): position
// rows of 256 fibers.  The chunk's coefficients (fwd, ip, g per position)
// are staged in shared memory.
template <typename R>
__device__ __forceinline__ void tp_stage_coef(R *sc, const ThomasTP<R> &t, uint32_t a) {
  for (uint32_t i = threadIdx.x; i < 4 * uint32_t(kTpC); i += blockDim.x)
    sc[i] = a + (i >> 2) < t.m ? t.q[4 * size_t(a) + i] : R(0);
}

// Load the lane's chunk (len positions) of fiber F into v.
template <typename R, int DIM>
__device__ __forceinline__ void tp_load(R (&v)[kTpC], const R *src, uint64_t F,
                                        uint32_t a, uint32_t len, uint32_t m0, uint32_t m1) {
  const uint64_t ps = tp_stride<DIM>(m0, m1);
  const R *p = src + tp_fiber_base<DIM>(F, m0, m1) + ps * a;
#pragma unroll
  for (int j = 0; j < kTpC; ++j)
    if (uint32_t(j) < len)
      v[j] = p[ps * j];
}

template <typename R, int DIM>
__global__ void __launch_bounds__(32 * kTpWarps, TP_MINB1)
    tp_pass1_kernel(const R *__restrict__ f, ThomasTP<R> t, uint64_t nfib, uint32_t m0,
                    uint32_t m1, R *__restrict__ E, R *__restrict__ S) {
  pdl_wait();
  __shared__ R sc[4 * kTpC];
  const uint32_t k = blockIdx.y, a = k * kTpC, len = min(uint32_t(kTpC), t.m - a);
  const uint64_t F = (uint64_t(blockIdx.x) * kTpWarps + (threadIdx.x >> 5)) * 32 +
                     (threadIdx.x & 31);
  R v[kTpC];
#pragma unroll
  for (int j = 0; j < kTpC; ++j)
    v[j] = R(0);
  // the fiber loads go out first; the coefficient staging overlaps them
  if (F < nfib)
    tp_load<R, DIM>(v, f, F, a, len, m0, m1);
  tp_stage_coef(sc, t, a);
  __syncthreads();
  if (F >= nfib)
    return;
  // forward from a zero carry (positions past len have zero coefficients
  // and values: they leave v at 0)
  R e = R(0);
#pragma unroll
  for (int j = 0; j < kTpC; ++j) {
    e = fma(sc[4 * j], e, v[j]);
    v[j] = e;
  }
  R eb = v[0]; // vl at the chunk's last real position
#pragma unroll
  for (int j = 1; j < kTpC; ++j)
    if (uint32_t(j) < len)
      eb = v[j];
  R x = R(0);
#pragma unroll
  for (int j = kTpC - 1; j >= 0; --j)
    x = fma(sc[4 * j + 2], x, sc[4 * j + 1] * v[j]);
  E[uint64_t(k) * nfib + F] = eb;
  S[uint64_t(k) * nfib + F] = x;
}

// CTA = 32 fibers (lane = fiber: every access is a coalesced row of the
// [chunk][fiber] scratch) x 32 warps; warp w owns the Q = ceil(K / 32) <= 16
// consecutive chunks [w*Q, w*Q + Q).  Forward: each thread composes its
// chunks' maps c -> PF c + E, the 32 warp maps meet in shared memory, each
// thread folds the maps of the warps below into its carry-in and replays
// its chunks (E[k] -> c_k).  Backward likewise with d -> PB d + (S + Q c)
// over the warps above (S[k] -> d_k).
constexpr int kTcWarps = 32;
constexpr int kTcQ = kTpMaxK / kTcWarps;
template <typename R>
__global__ void __launch_bounds__(32 * kTcWarps, 1)
    tp_carry_kernel(ThomasTP<R> t, uint64_t nfib, R *__restrict__ E, R *__restrict__ S) {
  pdl_wait();
  __shared__ R mA[kTcWarps][32], mB[kTcWarps][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t F = uint64_t(blockIdx.x) * 32 + lane;
  const bool ok = F < nfib;
  const uint64_t Fc = ok ? F : nfib - 1; // idle lanes shadow a real fiber (no stores)
  const uint32_t K = t.K, Q = (K + kTcWarps - 1) / kTcWarps, k0 = uint32_t(w) * Q;
  const uint32_t n = k0 < K ? min(Q, K - k0) : 0u;
  R x[kTcQ];
#pragma unroll
  for (int j = 0; j < kTcQ; ++j)
    if (uint32_t(j) < n)
      x[j] = E[uint64_t(k0 + j) * nfib + Fc];
  R A = R(1), B = R(0);
#pragma unroll
  for (int j = 0; j < kTcQ; ++j)
    if (uint32_t(j) < n) {
      const R pf = t.ck[4 * (k0 + j)];
      B = fma(pf, B, x[j]);
      A = pf * A;
    }
  mA[w][lane] = A;
  mB[w][lane] = B;
  __syncthreads();
  R c = R(0);
  for (int v = 0; v < w; ++v)
    c = fma(mA[v][lane], c, mB[v][lane]);
#pragma unroll
  for (int j = 0; j < kTcQ; ++j)
    if (uint32_t(j) < n) {
      const R e = x[j];
      x[j] = c; // c_k
      c = fma(t.ck[4 * (k0 + j)], c, e);
    }
  R y[kTcQ];
#pragma unroll
  for (int j = 0; j < kTcQ; ++j)
    if (uint32_t(j) < n) {
      if (ok)
        E[uint64_t(k0 + j) * nfib + F] = x[j];
      y[j] = S[uint64_t(k0 + j) * nfib + Fc];
    }
  __syncthreads(); // mA / mB reuse
  A = R(1);
  B = R(0);
#pragma unroll
  for (int j = kTcQ - 1; j >= 0; --j)
    if (uint32_t(j) < n) {
      const uint32_t k = k0 + j;
      y[j] = fma(t.ck[4 * k + 1], x[j], y[j]);
      const R pb = t.ck[4 * k + 2];
      B = fma(pb, B, y[j]);
      A = pb * A;
    }
  mA[w][lane] = A;
  mB[w][lane] = B;
  __syncthreads();
  R d = R(0);
  for (int v = kTcWarps - 1; v > w; --v)
    d = fma(mA[v][lane], d, mB[v][lane]);
#pragma unroll
  for (int j = kTcQ - 1; j >= 0; --j)
    if (uint32_t(j) < n) {
      const uint32_t k = k0 + j;
      if (ok)
        S[uint64_t(k) * nfib + F] = d;
      d = fma(t.ck[4 * k + 2], d, y[j]);
    }
}

template <typename R, int DIM>
__global__ void __launch_bounds__(32 * kTpWarps, TP_MINB2)
    tp_pass2_kernel(R *f, ThomasTP<R> t, uint64_t nfib, uint32_t m0, uint32_t m1,
                    const R *__restrict__ C, const R *__restrict__ D, Epi epi, const R *base,
                    R *out) {
  // f, base and out may alias (in-place apply: base == out; recompose: out == f);
  // every element is read and then written by the same thread only
  pdl_wait();
  __shared__ R sc[4 * kTpC];
  const uint32_t k = blockIdx.y, a = k * kTpC, len = min(uint32_t(kTpC), t.m - a);
  const uint64_t F = (uint64_t(blockIdx.x) * kTpWarps + (threadIdx.x >> 5)) * 32 +
                     (threadIdx.x & 31);
  R c = R(0), d = R(0);
  R v[kTpC], bs[kTpC];
#pragma unroll
  for (int j = 0; j < kTpC; ++j)
    v[j] = R(0);
  if (F < nfib) {
    c = C[uint64_t(k) * nfib + F];
    d = D[uint64_t(k) * nfib + F];
    tp_load<R, DIM>(v, f, F, a, len, m0, m1);
    // the epilogue bases go out with the fiber values (latency overlapped)
    if (epi != Epi::none)
      tp_load<R, DIM>(bs, base, F, a, len, m0, m1);
  }
  tp_stage_coef(sc, t, a);
  __syncthreads();
  if (F >= nfib)
    return;
  R e = c;
#pragma unroll
  for (int j = 0; j < kTpC; ++j) {
    e = fma(sc[4 * j], e, v[j]);
    v[j] = e;
  }
  // backward from d, injected at the chunk's last real position (padded
  // positions have g = ip = 0 and pass x = 0 down)
  R x = R(0);
#pragma unroll
  for (int j = kTpC - 1; j >= 0; --j) {
    const R xn = uint32_t(j) == len - 1 ? d : x;
    x = fma(sc[4 * j + 2], xn, sc[4 * j + 1] * v[j]);
    v[j] = x;
  }
  const uint64_t ps = tp_stride<DIM>(m0, m1);
  const uint64_t g0 = tp_fiber_base<DIM>(F, m0, m1) + ps * a;
  if (epi == Epi::none) {
#pragma unroll
    for (int j = 0; j < kTpC; ++j)
      if (uint32_t(j) < len)
        f[g0 + ps * j] = v[j];
  } else {
#pragma unroll
    for (int j = 0; j < kTpC; ++j)
      if (uint32_t(j) < len)
        out[g0 + ps * j] = epi == Epi::add ? bs[j] + v[j] : bs[j] - v[j];
  }
}

} // namespace mgrg
