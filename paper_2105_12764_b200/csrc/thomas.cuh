// thomas.cuh -- smem-resident batched Thomas solves (the IPK).
//
// thomas_fiber (/root/reference/proj/include/mgr/kernels.hpp:143-151):
//   forward   v_i += fwd_i * v_{i-1}          i = 1 .. m-1
//             v_{m-1} *= ip_{m-1}
//   backward  v_i = (v_i - h_i * v_{i+1}) * ip_i   i = m-2 .. 0
// is a serial recurrence per fiber; the reference evaluates it in exactly
// that order, so the bit-exact policy keeps one thread per fiber.  What the
// earlier kernels lost was the second HBM round trip: the forward results
// went back to global memory for the backward sweep.  Here a CTA stages
// whole fibers in shared memory, runs both sweeps there and writes each
// result once (with the apply / unapply epilogue of the level's last solve),
// so a solve costs one read and one write of the C-lattice -- the
// algorithmic minimum.  The sweeps are latency chains (FMUL->FADD, or one
// FFMA under the FAST policy); enough fibers resident per SM (3 CTAs x 32)
// hide them.
//
//   thomas_rows_kernel  fibers along dim 0: a CTA's 32 fibers are one
//                       contiguous chunk of 32*m elements (coalesced
//                       16-byte LDGSTS), pitch m in shared memory (odd m:
//                       conflict-free per-thread walks).
//   thomas_cols_kernel  fibers along dim 1 / 2 (stride S): a CTA's 32
//                       fibers are 32 adjacent inner positions, so every
//                       step of the staging is one 128-byte row; shared
//                       layout [m][32] is conflict-free.
#pragma once

#include "common.cuh"
#include "level.cuh"

namespace mgrg {

constexpr int kThomasFibers = 32;

template <typename R> __host__ __device__ constexpr uint32_t rows_pitch(uint32_t m) {
  return (m & 1u) ? m : m + 1; // odd pitch: lane t hits bank (t*pitch + i) % 32
}

template <typename R> constexpr size_t thomas_smem_limit() { return 200 * 1024; }

// Does the smem-resident path fit for fibers of length m?
template <typename R> __host__ inline bool thomas_resident_fits(uint32_t m) {
  return size_t(kThomasFibers) * rows_pitch<R>(m) * sizeof(R) <= thomas_smem_limit<R>();
}

template <typename R, bool FAST>
__device__ __forceinline__ R fwd_step(R x, R f, R v) {
  if constexpr (FAST)
    return fma(f, v, x);
  else
    return add(x, mul(f, v));
}
template <typename R, bool FAST>
__device__ __forceinline__ R bwd_step(R x, R h, R ip, R v) {
  if constexpr (FAST)
    return fma(-h, v, x) * ip;
  else
    return mul(sub(x, mul(h, v)), ip);
}

// One fiber in shared memory, element i at s[i * stride]: both sweeps in
// place.  fwd/h/ip are per-position (warp-uniform) loads.
template <typename R, bool FAST>
__device__ __forceinline__ void thomas_walk(R *s, uint32_t stride, const ThomasGeom<R> &t) {
  const uint32_t M = t.m;
  constexpr int U = 8;
  R v = s[0];
  uint32_t i = 1;
  for (; i + U <= M; i += U) {
    R x[U], fw[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      x[u] = s[(i + u) * stride];
      fw[u] = __ldg(t.fwd + i + u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v = fwd_step<R, FAST>(x[u], fw[u], v);
      s[(i + u) * stride] = v;
    }
  }
  for (; i < M; ++i) {
    v = fwd_step<R, FAST>(s[i * stride], __ldg(t.fwd + i), v);
    s[i * stride] = v;
  }
  v = mul(v, __ldg(t.ip + M - 1));
  s[(M - 1) * stride] = v;
  int32_t j = int32_t(M) - 2;
  for (; j - (U - 1) >= 0; j -= U) {
    R x[U], hh[U], pp[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      x[u] = s[(j - u) * stride];
      hh[u] = __ldg(t.h + j - u);
      pp[u] = __ldg(t.ip + j - u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v = bwd_step<R, FAST>(x[u], hh[u], pp[u], v);
      s[(j - u) * stride] = v;
    }
  }
  for (; j >= 0; --j) {
    v = bwd_step<R, FAST>(s[j * stride], __ldg(t.h + j), __ldg(t.ip + j), v);
    s[j * stride] = v;
  }
}

template <typename R>
__device__ __forceinline__ R epi_value(Epi epi, const R *base, uint64_t idx,
                                       R z) {
  if (epi == Epi::add)
    return add(base[idx], z); // apply_pack (refactor.hpp:388)
  if (epi == Epi::sub)
    return sub(base[idx], z); // unapply_expand (refactor.hpp:416)
  return z;
}

// ---------------------------------------------------------------------------
// dim 0: nfibers contiguous fibers of length m (fiber k at k*m).
// ---------------------------------------------------------------------------
template <typename R, bool FAST>
__global__ void __launch_bounds__(kThomasFibers)
    thomas_rows_kernel(R *f, ThomasGeom<R> t, uint64_t nfibers, Epi epi,
                       const R *base, R *out) {
  extern __shared__ __align__(16) unsigned char smem_bytes[];
  R *s = reinterpret_cast<R *>(smem_bytes);
  const uint32_t M = t.m, P = rows_pitch<R>(M);
  const int tid = threadIdx.x;
  const uint64_t fb0 = uint64_t(blockIdx.x) * kThomasFibers;
  const uint32_t nf = nfibers - fb0 < kThomasFibers ? uint32_t(nfibers - fb0) : kThomasFibers;
  const uint32_t total = nf * M;
  R *g = f + fb0 * M;
  // stage: fiber r element i -> s[r*P + i]
  if (P == M && (reinterpret_cast<uintptr_t>(g) & 15) == 0) {
    constexpr uint32_t V = 16 / sizeof(R);
    const uint32_t nv = total / V;
    for (uint32_t e = tid; e < nv; e += kThomasFibers)
      cp_async16(s + e * V, g + e * V);
    for (uint32_t e = nv * V + tid; e < total; e += kThomasFibers)
      cp_async(s + e, g + e);
  } else {
    for (uint32_t e = tid; e < total; e += kThomasFibers) {
      const uint32_t r = e / M, i = e - r * M;
      cp_async(s + r * P + i, g + e);
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
  if (uint32_t(tid) < nf)
    thomas_walk<R, FAST>(s + tid * P, 1, t);
  __syncwarp();
  R *o = (epi == Epi::none ? f : out) + fb0 * M;
  for (uint32_t e = tid; e < total; e += kThomasFibers) {
    const uint32_t r = e / M, i = e - r * M;
    o[e] = epi_value(epi, base, fb0 * M + e, s[r * P + i]);
  }
}

// ---------------------------------------------------------------------------
// dim 1 / 2: fiber k starts at (k % inner) + (k / inner) * ostride, element
// i at start + i*S.  32 consecutive fibers per CTA.
// ---------------------------------------------------------------------------
template <typename R, bool FAST>
__global__ void __launch_bounds__(kThomasFibers)
    thomas_cols_kernel(R *f, ThomasGeom<R> t, uint64_t S, uint64_t inner,
                       uint64_t ostride, uint64_t nfibers, Epi epi, const R *base,
                       R *out) {
  extern __shared__ __align__(16) unsigned char smem_bytes[];
  R *s = reinterpret_cast<R *>(smem_bytes);
  const uint32_t M = t.m;
  const int tid = threadIdx.x;
  const uint64_t k = uint64_t(blockIdx.x) * kThomasFibers + tid;
  const bool ok = k < nfibers;
  const uint64_t st = ok ? (k % inner) + (k / inner) * ostride : 0;
  if (ok) {
    const R *g = f + st;
    for (uint32_t i = 0; i < M; ++i)
      cp_async(s + i * kThomasFibers + tid, g + i * S);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
  if (!ok)
    return;
  // no cross-lane smem sharing: each lane owns its column
  thomas_walk<R, FAST>(s + tid, kThomasFibers, t);
  R *o = epi == Epi::none ? f : out;
  for (uint32_t i = 0; i < M; ++i)
    o[st + i * S] = epi_value(epi, base, st + i * S, s[i * kThomasFibers + tid]);
}

template <typename R> __host__ inline size_t thomas_rows_smem(uint32_t m) {
  return size_t(kThomasFibers) * rows_pitch<R>(m) * sizeof(R);
}
template <typename R> __host__ inline size_t thomas_cols_smem(uint32_t m) {
  return size_t(kThomasFibers) * m * sizeof(R);
}

} // namespace mgrg
