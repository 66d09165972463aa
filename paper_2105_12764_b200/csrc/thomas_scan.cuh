// thomas_scan.cuh -- warp-parallel Thomas solves for the FAST policy.
//
// Both sweeps of thomas_fiber (/root/reference/proj/include/mgr/kernels.hpp
// :143-151) are first-order linear recurrences:
//   forward   v_i = x_i + a_i v_{i-1}           (a_i = fwd_i, a_0 = 0)
//   backward  z_i = c_i + d_i z_{i+1}            (c_i = ip_i v_i, d_i = -h_i ip_i)
// so a fiber can be split over the 32 lanes of a warp: every lane reduces
// its contiguous segment to an affine map, a 5-step shuffle scan composes
// the maps, and each lane replays its segment from the exact incoming value.
// The operator is the reference's; only the association of the recurrence
// changes (the FAST policy's tolerance, not bit-exactness -- the exact
// policy keeps thomas.cuh's one-thread-per-fiber walk).  With the whole
// warp on one fiber, occupancy no longer depends on how many fibers fit in
// shared memory, and each solve is one HBM read and one write.
//
//   thomas_scan_rows_kernel  fibers along dim 0 (contiguous): a warp
//       stages one fiber with coalesced LDGSTS into a warp-private buffer,
//       lanes take segments of S = ceil(m/32) (odd S: conflict-free).
//   thomas_scan_cols_kernel  fibers along dim 1 (stride S): a CTA stages a
//       [m][33] tile of 32 adjacent fibers (128-byte rows), eight warps scan
//       four fibers each.
#pragma once

#include "common.cuh"
#include "level.cuh"

namespace mgrg {

__host__ __device__ constexpr uint32_t scan_seg(uint32_t m) {
  const uint32_t s = (m + 31) / 32;
  return s | 1u; // odd segment length: lane l's element i at bank (s*l + i)
}

// Per-position coefficients staged once per CTA: a (fwd), ip, d = -h*ip.
template <typename R>
__device__ __forceinline__ void stage_coef(R *ca, R *cip, R *cd, const ThomasGeom<R> &t) {
  for (uint32_t i = threadIdx.x; i < t.m; i += blockDim.x) {
    ca[i] = t.fwd[i];
    const R ip = t.ip[i];
    cip[i] = ip;
    cd[i] = i + 1 < t.m ? -t.h[i] * ip : R(0);
  }
}

// Solve one fiber held in smem, element i at s[i * st]; lane segments of
// length SEG.  In place.
template <typename R, uint32_t SEGMAX>
__device__ __forceinline__ void scan_solve(R *s, uint32_t st, uint32_t m, uint32_t seg,
                                           const R *ca, const R *cip, const R *cd,
                                           int lane) {
  const uint32_t i0 = seg * lane;
  const uint32_t i1 = min(i0 + seg, m);
  R x[SEGMAX];
  // ---- forward: local map (A, B) over the segment
  R A = R(1), B = R(0);
#pragma unroll
  for (uint32_t k = 0; k < SEGMAX; ++k) {
    const uint32_t i = i0 + k;
    if (i < i1) {
      x[k] = s[i * st];
      const R a = ca[i];
      B = fma(a, B, x[k]);
      A = A * a;
    }
  }
  // inclusive scan of maps: lane l gets the map of lanes 0..l
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const R pA = __shfl_up_sync(0xffffffffu, A, d);
    const R pB = __shfl_up_sync(0xffffffffu, B, d);
    if (lane >= d) {
      B = fma(A, pB, B);
      A = A * pA;
    }
  }
  R v = __shfl_up_sync(0xffffffffu, B, 1); // value before the segment
  if (lane == 0)
    v = R(0);
  // replay the segment; the last element takes its pivot: v_{m-1} *= ip
#pragma unroll
  for (uint32_t k = 0; k < SEGMAX; ++k) {
    const uint32_t i = i0 + k;
    if (i < i1) {
      v = fma(ca[i], v, x[k]);
      x[k] = i + 1 == m ? v * cip[i] : v;
    }
  }
  // ---- backward: z_i = c_i + d_i z_{i+1}, c_i = ip_i v_i (z_{m-1} = x_{m-1})
  A = R(1);
  B = R(0);
#pragma unroll
  for (int k = SEGMAX - 1; k >= 0; --k) {
    const uint32_t i = i0 + k;
    if (i < i1) {
      const R c = i + 1 == m ? x[k] : x[k] * cip[i];
      const R d = cd[i];
      B = fma(d, B, c);
      A = A * d;
    }
  }
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const R nA = __shfl_down_sync(0xffffffffu, A, d);
    const R nB = __shfl_down_sync(0xffffffffu, B, d);
    if (lane + d < 32) {
      B = fma(A, nB, B);
      A = A * nA;
    }
  }
  R z = __shfl_down_sync(0xffffffffu, B, 1); // value after the segment
  if (lane == 31)
    z = R(0);
#pragma unroll
  for (int k = SEGMAX - 1; k >= 0; --k) {
    const uint32_t i = i0 + k;
    if (i < i1) {
      const R c = i + 1 == m ? x[k] : x[k] * cip[i];
      z = fma(cd[i], z, c);
      s[i * st] = z;
    }
  }
}

template <typename R>
__device__ __forceinline__ R epi_apply(Epi epi, const R *base, uint64_t idx, R z) {
  if (epi == Epi::add)
    return add(base[idx], z);
  if (epi == Epi::sub)
    return sub(base[idx], z);
  return z;
}

// ---------------------------------------------------------------------------
// dim 0: nfibers contiguous fibers of length m; warp per fiber.
// ---------------------------------------------------------------------------
template <typename R, uint32_t SEGMAX>
__global__ void __launch_bounds__(256)
    thomas_scan_rows_kernel(R *f, ThomasGeom<R> t, uint64_t nfibers, Epi epi,
                            const R *base, R *out) {
  extern __shared__ __align__(16) unsigned char smem_bytes[];
  const uint32_t m = t.m, seg = scan_seg(m), pitch = 32 * seg;
  R *ca = reinterpret_cast<R *>(smem_bytes);
  R *cip = ca + m;
  R *cd = cip + m;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  R *buf = cd + m + ((3 * m) & 1) + warp * pitch; // keep 8-byte alignment for f64 math
  stage_coef(ca, cip, cd, t);
  __syncthreads();
  const uint64_t stride = uint64_t(gridDim.x) * 8;
  for (uint64_t k = uint64_t(blockIdx.x) * 8 + warp; k < nfibers; k += stride) {
    const R *g = f + k * m;
    for (uint32_t i = lane; i < m; i += 32)
      cp_async(buf + i, g + i);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
    scan_solve<R, SEGMAX>(buf, 1, m, seg, ca, cip, cd, lane);
    __syncwarp();
    R *o = (epi == Epi::none ? f : out) + k * m;
    for (uint32_t i = lane; i < m; i += 32)
      o[i] = epi_apply(epi, base, k * m + i, buf[i]);
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// dim 1 (and dim 2 when the caller chooses): fiber k starts at
// (k % inner) + (k / inner) * ostride, element i at start + i*S.  32
// consecutive fibers per CTA, 8 warps x 4 fibers.
// ---------------------------------------------------------------------------
template <typename R, uint32_t SEGMAX>
__global__ void __launch_bounds__(256)
    thomas_scan_cols_kernel(R *f, ThomasGeom<R> t, uint64_t S, uint64_t inner,
                            uint64_t ostride, uint64_t nfibers, Epi epi, const R *base,
                            R *out) {
  extern __shared__ __align__(16) unsigned char smem_bytes[];
  const uint32_t m = t.m, seg = scan_seg(m);
  R *ca = reinterpret_cast<R *>(smem_bytes);
  R *cip = ca + m;
  R *cd = cip + m;
  R *tile = cd + m + ((3 * m) & 1); // [m][33]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  stage_coef(ca, cip, cd, t);
  // stage: row i (element i of the 32 fibers) -> tile[i*33 + col]
  const uint64_t k = uint64_t(blockIdx.x) * 32 + lane;
  const bool ok = k < nfibers;
  const uint64_t st = ok ? (k % inner) + (k / inner) * ostride : 0;
  if (ok)
    for (uint32_t i = warp; i < m; i += 8)
      cp_async(tile + i * 33 + lane, f + st + i * S);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll 1
  for (int c = 0; c < 4; ++c) {
    const int col = warp * 4 + c;
    if (uint64_t(blockIdx.x) * 32 + col < nfibers)
      scan_solve<R, SEGMAX>(tile + col, 33, m, seg, ca, cip, cd, lane);
  }
  __syncthreads();
  R *o = epi == Epi::none ? f : out;
  if (ok)
    for (uint32_t i = warp; i < m; i += 8)
      o[st + i * S] = epi_apply(epi, base, st + i * S, tile[i * 33 + lane]);
}

template <typename R> __host__ inline size_t scan_rows_smem(uint32_t m) {
  return sizeof(R) * (3 * m + 1 + 8 * 32 * size_t(scan_seg(m)));
}
template <typename R> __host__ inline size_t scan_cols_smem(uint32_t m) {
  return sizeof(R) * (3 * m + 1 + 33 * size_t(m));
}

} // namespace mgrg
