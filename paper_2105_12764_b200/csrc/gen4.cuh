// gen4.cuh -- 4-D levels (spatiotemporal grids).
//
// The 3-D family (lean.cuh, kernels*.cuh) is tiled for three dimensions;
// a fourth (the stacked time axis of decompose_spatiotemporal,
// refactor.hpp:536-567) goes through this generic path instead.  Every
// step of a level is one element-parallel pass over a compact lattice:
//
//   decompose  coef   : W = u - interp(u) at nodes fine in any dim, 0 at
//                       all-coarse nodes (gpk_sweep + the vec(C) mask of
//                       masstrans_dim0, refactor.hpp:251-307), fused with
//                       the class store (class_slot, grid.hpp:149-164)
//              mass d : W (dims < d coarse, dims >= d fine) -> R*M along d
//                       (masstrans_window, kernels.hpp:158-185); one pass per
//                       dimension that refines, ping-pong between buffers
//              solve d: Thomas along d on the coarse lattice
//                       (thomas_fiber, kernels.hpp:143-151), in place, with
//                       the 3-D family's exact-order Thomas kernels
//              apply  : a_{l-1}[i] = a_l[off(i)] + z[i]  (refactor.hpp:380-399)
//   recompose  load   : W = class value at fine nodes, 0 elsewhere
//              mass/solve as above, then a' = a_{l-1} - z  (refactor.hpp:404-422)
//              rgpk   : out = a' at coarse nodes, interp(a') + class at fine
//                       nodes (scatter_class + inverse gpk_sweep)
//
// All arithmetic is the reference expression through the _rn intrinsics, so
// both policies are bit-identical to the reference on 4-D grids (the FAST
// tolerance is met trivially).  The lattices are compact and dim-0-fastest,
// so each pass reads and writes unit-stride along dim 0.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace mgrg {

constexpr int kGenDims = 4;

// Division by a fixed extent as a multiply-high (the decode of a flat index
// is the element-parallel kernels' main cost: three 32-bit divisions by
// runtime divisors are ~60 instructions, these ~12): with l = ceil(log2 d),
// m = floor(2^32 (2^l - d) / d) + 1, n / d = (t + ((n - t) >> 1)) >> (l - 1),
// t = umulhi(m, n), exact for every 32-bit n (d = 1: identity).
struct FastDiv {
  uint32_t d, m, sh;
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0u, 0u};
  if (d > 1) {
    uint32_t l = 0;
    while ((uint64_t(1) << l) < d)
      ++l;
    f.m = uint32_t(((uint64_t(1) << 32) * ((uint64_t(1) << l) - d)) / d + 1);
    f.sh = l - 1;
  }
  return f;
}
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv &f) {
  if (f.d == 1)
    return n;
  const uint32_t t = __umulhi(f.m, n);
  return (t + ((n - t) >> 1)) >> f.sh;
}

template <typename R> struct Gen4Geom {
  uint32_t n[kGenDims];            // level-l extents
  uint32_t m[kGenDims];            // level-(l-1) extents
  FastDiv fn[kGenDims], fm[kGenDims]; // their fast divisors
  const R *h[kGenDims];            // level-l spacings (grid.cpp:60-65)
  const R *r[kGenDims];            // level-l ratios (grid.cpp:66-71)
  const R *th[kGenDims];           // level-(l-1) Thomas factors (kernels.hpp:107-135),
  const R *tf[kGenDims];           // null where the dimension does not refine
  const R *ti[kGenDims];
  uint64_t tbase[1 << kGenDims];   // class type bases (grid.cpp:151-162)
  uint32_t cext[1 << kGenDims][kGenDims]; // class type extents

  __host__ __device__ uint64_t nodes() const {
    return uint64_t(n[0]) * n[1] * n[2] * n[3];
  }
  __host__ __device__ uint64_t coarse_nodes() const {
    return uint64_t(m[0]) * m[1] * m[2] * m[3];
  }
};

// flat index -> lattice position with fast divisors (32-bit indices)
__device__ __forceinline__ void gen_decode_f(uint64_t i, const FastDiv *f, uint32_t *p) {
  if ((i >> 32) == 0) {
    uint32_t j = uint32_t(i);
#pragma unroll
    for (int d = 0; d < kGenDims - 1; ++d) {
      const uint32_t qd = fdiv(j, f[d]);
      p[d] = j - qd * f[d].d;
      j = qd;
    }
    p[kGenDims - 1] = j;
    return;
  }
#pragma unroll
  for (int d = 0; d < kGenDims; ++d) {
    p[d] = uint32_t(i % f[d].d);
    i /= f[d].d;
  }
}

template <typename R>
__device__ __forceinline__ unsigned gen_mask(const Gen4Geom<R> &g, const uint32_t *p) {
  unsigned mask = 0;
#pragma unroll
  for (int d = 0; d < kGenDims; ++d)
    if (!is_coarse(p[d], g.n[d]))
      mask |= 1u << d;
  return mask;
}

// class_slot (grid.hpp:149-164)
template <typename R>
__device__ __forceinline__ uint64_t gen_slot(const Gen4Geom<R> &g, const uint32_t *p,
                                             unsigned mask) {
  uint64_t idx = 0, mult = 1;
#pragma unroll
  for (int d = 0; d < kGenDims; ++d) {
    const uint32_t w = ((mask >> d) & 1) ? fine_rank(p[d]) : coarse_rank(p[d]);
    idx += w * mult;
    mult *= g.cext[mask][d];
  }
  return g.tbase[mask] + idx;
}

// interpolate_node (kernels.hpp:193-223): corners at p +- 1 along the fine
// dims, reduced pairwise a + t*(b - a), lowest fine dim first.  Corner c
// carries bit d for dimension d (all four, statically indexed: no local
// memory); only the 2^k corners of the k fine dims are loaded, and a
// non-fine dimension's reduction step keeps the even corner unchanged, which
// pairs and orders the lerps exactly like the reference's compacted corner
// index.  `at(q)` reads the level-l value at lattice position q.
template <typename R, typename At>
__device__ __forceinline__ R gen_interp(const Gen4Geom<R> &g, const uint32_t *p, unsigned mask,
                                        At &&at) {
  R c[1 << kGenDims];
#pragma unroll
  for (int ci = 0; ci < (1 << kGenDims); ++ci) {
    c[ci] = R(0);
    if ((unsigned(ci) & ~mask) == 0) {
      uint32_t q[kGenDims];
#pragma unroll
      for (int d = 0; d < kGenDims; ++d)
        q[d] = ((mask >> d) & 1) ? (((ci >> d) & 1) ? p[d] + 1 : p[d] - 1) : p[d];
      c[ci] = at(q);
    }
  }
#pragma unroll
  for (int d = 0; d < kGenDims; ++d) {
    const bool fine = (mask >> d) & 1;
    const R t = fine ? g.r[d][p[d] - 1] : R(0);
#pragma unroll
    for (int i = 0; i < ((1 << kGenDims) >> (d + 1)); ++i)
      c[i] = fine ? lerp(c[2 * i], c[2 * i + 1], t) : c[2 * i];
  }
  return c[0];
}

template <typename R>
__device__ __forceinline__ uint64_t gen_lattice_off(const Gen4Geom<R> &g, const uint32_t *q) {
  return q[0] + uint64_t(g.n[0]) * (q[1] + uint64_t(g.n[1]) * (q[2] + uint64_t(g.n[2]) * q[3]));
}

// decompose: coefficients + vec(C) field + class store
template <typename R>
__global__ void gen_coef_kernel(Gen4Geom<R> g, const R *__restrict__ a, R *__restrict__ W,
                                R *__restrict__ cls) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= g.nodes())
    return;
  uint32_t p[kGenDims];
  gen_decode_f(i, g.fn, p);
  const unsigned mask = gen_mask(g, p);
  if (!mask) {
    W[i] = R(0);
    return;
  }
  const R ip = gen_interp(g, p, mask, [&](const uint32_t *q) { return a[gen_lattice_off(g, q)]; });
  const R coef = sub(a[i], ip);
  W[i] = coef;
  cls[gen_slot(g, p, mask)] = coef;
}

// recompose: vec(C) field from the class (null class = zeros)
template <typename R>
__global__ void gen_load_kernel(Gen4Geom<R> g, const R *__restrict__ cls, R *__restrict__ W) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= g.nodes())
    return;
  uint32_t p[kGenDims];
  gen_decode_f(i, g.fn, p);
  const unsigned mask = gen_mask(g, p);
  W[i] = (mask && cls) ? cls[gen_slot(g, p, mask)] : R(0);
}

// R*M along dim d: input extents e (e[d] = n[d]), output extents e with
// e[d] = m[d]; one thread per output node
template <typename R>
__global__ void gen_mass_kernel(Gen4Geom<R> g, int d, uint4 e4, const R *__restrict__ in,
                                R *__restrict__ out) {
  const uint32_t e[kGenDims] = {e4.x, e4.y, e4.z, e4.w};
  uint32_t oe[kGenDims] = {e4.x, e4.y, e4.z, e4.w};
  const uint32_t n = g.n[d];
  oe[d] = g.m[d];
  const uint64_t total = uint64_t(oe[0]) * oe[1] * oe[2] * oe[3];
  const uint64_t o = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (o >= total)
    return;
  uint32_t p[kGenDims];
  // output extents: dims <= d at level l-1, dims > d at level l
  FastDiv fo[kGenDims];
#pragma unroll
  for (int k = 0; k < kGenDims; ++k)
    fo[k] = k <= d ? g.fm[k] : g.fn[k];
  gen_decode_f(o, fo, p);
  uint64_t base = 0, str = 1, sd = 1;
#pragma unroll
  for (int k = 0; k < kGenDims; ++k) {
    if (k == d)
      sd = str;
    else
      base += p[k] * str;
    str *= e[k];
  }
  const uint32_t q = coarse_pos(p[d], n);
  out[o] = masstrans_at<R>([&](uint32_t j) { return in[base + j * sd]; }, q, n, g.h[d], g.r[d]);
}

// decompose apply_pack: P[i] = a[off(i)] + z[i]
template <typename R>
__global__ void gen_apply_kernel(Gen4Geom<R> g, const R *__restrict__ a,
                                 const R *__restrict__ z, R *__restrict__ P) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= g.coarse_nodes())
    return;
  uint32_t c[kGenDims], q[kGenDims];
  gen_decode_f(i, g.fm, c);
#pragma unroll
  for (int d = 0; d < kGenDims; ++d)
    q[d] = coarse_pos(c[d], g.n[d]);
  P[i] = add(a[gen_lattice_off(g, q)], z[i]);
}

// recompose unapply_expand on the compact coarse lattice: z <- prev - z
template <typename R>
__global__ void gen_unapply_kernel(uint64_t count, const R *__restrict__ prev, R *__restrict__ z) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < count)
    z[i] = sub(prev[i], z[i]);
}

// recompose: scatter_class + inverse gpk_sweep from the corrected coarse
// lattice cz (compact, level-(l-1) extents)
template <typename R>
__global__ void gen_rgpk_kernel(Gen4Geom<R> g, const R *__restrict__ cz,
                                const R *__restrict__ cls, R *__restrict__ out) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= g.nodes())
    return;
  uint32_t p[kGenDims];
  gen_decode_f(i, g.fn, p);
  const unsigned mask = gen_mask(g, p);
  auto at = [&](const uint32_t *q) {
    return cz[coarse_rank(q[0]) +
              uint64_t(g.m[0]) * (coarse_rank(q[1]) +
                                  uint64_t(g.m[1]) * (coarse_rank(q[2]) +
                                                      uint64_t(g.m[2]) * coarse_rank(q[3])))];
  };
  if (!mask) {
    out[i] = at(p);
    return;
  }
  const R ip = gen_interp(g, p, mask, at);
  out[i] = add(ip, cls ? cls[gen_slot(g, p, mask)] : R(0));
}

// unit-level compute_coefficients / restore_coefficients in place
// (kernels.hpp:284-310): corners are coarse nodes, never written
template <typename R>
__global__ void gen_gpk_inplace_kernel(Gen4Geom<R> g, R *a, int inverse) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= g.nodes())
    return;
  uint32_t p[kGenDims];
  gen_decode_f(i, g.fn, p);
  const unsigned mask = gen_mask(g, p);
  if (!mask)
    return;
  const R ip = gen_interp(g, p, mask, [&](const uint32_t *q) { return a[gen_lattice_off(g, q)]; });
  a[i] = inverse ? add(ip, a[i]) : sub(a[i], ip);
}

// unit-level masstrans_apply along dim 0 (kernels.hpp:328-412): the vec(C)
// input (all-coarse nodes as 0) and the optional fused class copy
template <typename R>
__global__ void gen_vecc_kernel(Gen4Geom<R> g, const R *__restrict__ in, R *__restrict__ W,
                                R *__restrict__ coef) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= g.nodes())
    return;
  uint32_t p[kGenDims];
  gen_decode_f(i, g.fn, p);
  const unsigned mask = gen_mask(g, p);
  const R x = in[i];
  W[i] = mask ? x : R(0);
  if (mask && coef)
    coef[gen_slot(g, p, mask)] = x;
}

// reorder / to_natural (grid.hpp:177-196): coarse-first index of natural
// node i is its coarse rank (all-coarse nodes) or C + its class slot
template <typename R>
__global__ void gen_reorder_kernel(Gen4Geom<R> g, int to_natural, const R *__restrict__ in,
                                   R *__restrict__ out) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= g.nodes())
    return;
  uint32_t p[kGenDims];
  gen_decode_f(i, g.fn, p);
  const unsigned mask = gen_mask(g, p);
  const uint64_t k =
      mask ? g.coarse_nodes() + gen_slot(g, p, mask)
           : coarse_rank(p[0]) +
                 uint64_t(g.m[0]) * (coarse_rank(p[1]) +
                                     uint64_t(g.m[1]) * (coarse_rank(p[2]) +
                                                         uint64_t(g.m[2]) * coarse_rank(p[3])));
  if (to_natural)
    out[i] = in[k];
  else
    out[k] = in[i];
}

} // namespace mgrg
