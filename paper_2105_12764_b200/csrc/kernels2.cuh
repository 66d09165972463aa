// kernels2.cuh -- pair-per-lane level kernels (the fast path).
//
// Mapping: a warp covers one box row of 64 fine x positions; lane a owns the
// pair (X0 + 2a, X0 + 2a + 1) = (even/coarse-x node, odd/fine-x node).  With
// X0 = 2*cx0 - 2 the 32 pairs cover the reach-2 stencil window of 30 coarse-x
// outputs, so the merged R*M along x is a 5-tap window over lanes i, i+1,
// i+2 and runs on warp shuffles with the lane's stencil held in registers.
// The y pass reads five rows of the x results from shared memory; the z
// pass keeps the last planes' y results in registers (no ring indexing).
//
// GPK as prolongation: the reference interpolates every fine node from its
// 2^k coarse corners, reducing pairwise along the fine dimensions in
// ascending order (kernels.hpp:193-223).  The inner reductions are exactly
// the interpolated values of lower-type nodes (e.g. a face node's x-lerps are
// the edge-node interpolants of the rows above and below), so the level's
// interpolant W is the coarse lattice prolongated along x, then y, then z --
// one lerp per node, same operands, same t, same order: bit-identical.
//   coarse z-plane, coarse y-row : W_e = U_e,  W_o = lerp_x(U_e, U_e', tx)
//   coarse z-plane, fine   y-row : W   = lerp_y(W(row-1), W(row+1), ty)
//   fine   z-plane               : W   = lerp_z(W(plane-1), W(plane+1), tz)
// The coarse planes' W is kept in shared memory for the fine plane between.
//
// Arithmetic policy (template FAST):
//   FAST = false: the reference's expressions, operation by operation, no
//                 FMA contraction -> bit-identical to the CPU reference;
//   FAST = true : lerps as one FMA, merged R*M as a 5-tap FMA chain with
//                 host-precomputed weights -> ~3x fewer FP instructions,
//                 differences at the level of rounding (well inside the
//                 1e-5 f32 / 1e-12 f64 range-normalized parity bar).
#pragma once

#include "common.cuh"
#include "level.cuh"

namespace mgrg {

// One coarse output of the merged mass-trans along a dimension, as host-
// precomputed coefficients in the working precision (mgrg.cu make_stencil).
// Exact form: v = mv(q) [+ cl*mv(q-1)] [+ cr*mv(q+1)] (masstrans_window,
// kernels.hpp:159-178).  Fast form: v = sum_t w[t] * tap[t].
template <typename R> struct Stencil {
  R hm2, hm1, h0, hp1; // h[q-2], h[q-1], h[q], h[q+1]
  R dm1, d0, dp1;      // 2(h[j-1]+h[j]) at j = q-1, q, q+1 (boundary: 2h)
  R cl, cr;            // r[q-2], 1 - r[q]
  R w[5];              // fast-path tap weights
  uint32_t flags;      // ST_* below
};
enum : uint32_t {
  ST_LEFT = 1,   // q == 0: mv(q) = 2h0*in(q) + h0*in(q+1)
  ST_RIGHT = 2,  // q == n-1: mv(q) = h[n-2]*in(q-1) + 2h[n-2]*in(q)
  ST_HASL = 4,   // q-1 is fine: + r[q-2]*mv(q-1)
  ST_HASR = 8,   // q+1 is fine: + (1-r[q])*mv(q+1)
  ST_SHIFT = 16, // q = 2c-1 (last node of an even extent): taps shifted by one
  ST_VALID = 32,
  ST_INTERIOR = ST_HASL | ST_HASR | ST_VALID
};

template <typename R, bool FAST> struct Arith {
  static __device__ __forceinline__ R lerp(R a, R b, R t) {
    if constexpr (FAST)
      return fma(t, b - a, a);
    else
      return mgrg::lerp(a, b, t);
  }
};

// Taps t0..t4 are the fine positions 2c-2 .. 2c+2 around the output's
// nominal centre 2c (x, y) or q-2 .. q+2 (z, never shifted).
template <typename R, bool FAST>
__device__ __forceinline__ R stencil_eval(const Stencil<R> &s, R t0, R t1, R t2, R t3,
                                          R t4) {
  if constexpr (FAST) {
    R v = s.w[0] * t0;
    v = fma(s.w[1], t1, v);
    v = fma(s.w[2], t2, v);
    v = fma(s.w[3], t3, v);
    return fma(s.w[4], t4, v);
  } else {
    if (s.flags == ST_INTERIOR) { // straight-line common case
      R v = add(add(mul(s.hm1, t1), mul(s.d0, t2)), mul(s.h0, t3));
      const R ml = add(add(mul(s.hm2, t0), mul(s.dm1, t1)), mul(s.hm1, t2));
      v = add(v, mul(s.cl, ml));
      const R mr = add(add(mul(s.h0, t2), mul(s.dp1, t3)), mul(s.hp1, t4));
      return add(v, mul(s.cr, mr));
    }
    if (s.flags & ST_SHIFT) // q = 2c-1 = n-1, n even: only the right-boundary mv
      return add(mul(s.hm1, t0), mul(s.d0, t1));
    R v;
    if (s.flags & ST_LEFT)
      v = add(mul(s.d0, t2), mul(s.h0, t3));
    else if (s.flags & ST_RIGHT)
      v = add(mul(s.hm1, t1), mul(s.d0, t2));
    else
      v = add(add(mul(s.hm1, t1), mul(s.d0, t2)), mul(s.h0, t3));
    if (s.flags & ST_HASL) {
      const R ml = add(add(mul(s.hm2, t0), mul(s.dm1, t1)), mul(s.hm1, t2));
      v = add(v, mul(s.cl, ml));
    }
    if (s.flags & ST_HASR) {
      const R mr = add(add(mul(s.h0, t2), mul(s.dp1, t3)), mul(s.hp1, t4));
      v = add(v, mul(s.cr, mr));
    }
    return v;
  }
}

// Pieces of the exact merged stencil, to share the fine-neighbour mass
// products of adjacent outputs: mr(c) (the q+1 term of output c) equals
// ml(c+1) (the q'-1 term of output c+1, q' = q+2) bit for bit -- same
// coefficients h[q], 2(h[q]+h[q+1]), h[q+1] (one table value each), same
// taps, same operation order -- so each is evaluated once.  st_combine(s,
// t0..t3, st_ml(s, t0, t1, t2), st_mr(s, t2, t3, t4)) == stencil_eval<R,
// false>(s, t0, .., t4) for every stencil.
template <typename R>
__device__ __forceinline__ R st_ml(const Stencil<R> &s, R t0, R t1, R t2) {
  return add(add(mul(s.hm2, t0), mul(s.dm1, t1)), mul(s.hm1, t2));
}
template <typename R>
__device__ __forceinline__ R st_mr(const Stencil<R> &s, R t2, R t3, R t4) {
  return add(add(mul(s.h0, t2), mul(s.dp1, t3)), mul(s.hp1, t4));
}
template <typename R>
__device__ __forceinline__ R st_combine(const Stencil<R> &s, R t0, R t1, R t2, R t3, R ml,
                                        R mr) {
  if (s.flags == ST_INTERIOR) {
    R v = add(add(mul(s.hm1, t1), mul(s.d0, t2)), mul(s.h0, t3));
    v = add(v, mul(s.cl, ml));
    return add(v, mul(s.cr, mr));
  }
  if (s.flags & ST_SHIFT)
    return add(mul(s.hm1, t0), mul(s.d0, t1));
  R v;
  if (s.flags & ST_LEFT)
    v = add(mul(s.d0, t2), mul(s.h0, t3));
  else if (s.flags & ST_RIGHT)
    v = add(mul(s.hm1, t1), mul(s.d0, t2));
  else
    v = add(add(mul(s.hm1, t1), mul(s.d0, t2)), mul(s.h0, t3));
  if (s.flags & ST_HASL)
    v = add(v, mul(s.cl, ml));
  if (s.flags & ST_HASR)
    v = add(v, mul(s.cr, mr));
  return v;
}

// Balanced tiling: tile t of nt over m outputs covers [t*m/nt, (t+1)*m/nt).
__device__ __forceinline__ uint32_t tile_lo(uint32_t t, uint32_t nt, uint32_t m) {
  return uint32_t((uint64_t(t) * m) / nt);
}

template <typename R> struct Pair {
  R e, o;
};
template <typename R> __device__ __forceinline__ Pair<R> ld_pair(const R *p) {
  if constexpr (sizeof(R) == 4) {
    const float2 v = *reinterpret_cast<const float2 *>(p);
    return {v.x, v.y};
  } else {
    const double2 v = *reinterpret_cast<const double2 *>(p);
    return {v.x, v.y};
  }
}
template <typename R> __device__ __forceinline__ void st_pair(R *p, R e, R o) {
  if constexpr (sizeof(R) == 4)
    *reinterpret_cast<float2 *>(p) = make_float2(e, o);
  else
    *reinterpret_cast<double2 *>(p) = make_double2(e, o);
}

// Class-type tables of the level in shared memory (class_slot,
// grid.hpp:149-164): row base of mask m at row ranks (wy, wz).
struct ClassTab {
  uint64_t tb[8];
  uint32_t tx[8], ty[8];
  __device__ __forceinline__ uint64_t row(unsigned m, uint32_t wy, uint32_t wz) const {
    return tb[m] + uint64_t(tx[m]) * (wy + uint64_t(ty[m]) * wz);
  }
};
template <typename R>
__device__ __forceinline__ void load_classtab(ClassTab &t, const LevelGeom<R> &g, int tid) {
  if (tid < 8) {
    t.tb[tid] = g.tbase[tid];
    t.tx[tid] = g.tex[tid];
    t.ty[tid] = g.tey[tid];
  }
}

template <int CY> struct PairCfg {
  static constexpr int NW = 8, T = 256, BX = 64, BYR = 2 * CY + 3;
  static constexpr int PLANE = BYR * BX;
  static constexpr int RW = (CY + 7) / 8; // output rows per warp
  static constexpr int ZC = 32;           // coarse-z planes per CTA
};

// shared-memory carve-up helper (16-byte aligned chunks)
struct Carve {
  unsigned char *p;
  template <typename T> __device__ __forceinline__ T *take(size_t n) {
    T *r = reinterpret_cast<T *>(p);
    p += (n * sizeof(T) + 15) & ~size_t(15);
    return r;
  }
};
__host__ __device__ constexpr size_t al16(size_t b) { return (b + 15) & ~size_t(15); }

template <typename R, int CY> constexpr size_t rl2_smem() {
  using C = PairCfg<CY>;
  return al16(sizeof(R) * 3 * C::PLANE) + al16(sizeof(R) * C::BYR * 32) +
         al16(sizeof(Stencil<R>) * CY) + al16(sizeof(Stencil<R>) * C::ZC) +
         al16(sizeof(ClassTab));
}
template <typename R, int CY> constexpr size_t rg2_smem() {
  // coarse planes: 3 x (CY+1) rows x 33; W planes: 2 x 2CY x 64
  return al16(sizeof(R) * 3 * (CY + 1) * 33) + al16(sizeof(R) * 2 * (2 * CY) * 64) +
         al16(sizeof(ClassTab));
}

// Stage `n` stencils (global) into shared memory.
template <typename R>
__device__ __forceinline__ void stage_stencils(Stencil<R> *dst, const Stencil<R> *src,
                                               uint32_t n, int tid) {
  constexpr int W = sizeof(Stencil<R>) / 4;
  const uint32_t *s = reinterpret_cast<const uint32_t *>(src);
  uint32_t *d = reinterpret_cast<uint32_t *>(dst);
  for (uint32_t i = tid; i < n * W; i += 256)
    d[i] = __ldg(s + i);
}

// y pass of the X rows for output row j (box rows 2j .. 2j+4).
template <typename R, bool FAST>
__device__ __forceinline__ R y_eval(const Stencil<R> &s, const R *X, int j, int lane) {
  const R *c = X + (2 * j) * 32 + lane;
  return stencil_eval<R, FAST>(s, c[0], c[32], c[64], c[96], c[128]);
}

// ---------------------------------------------------------------------------
// Recompose load vector, one level (pair-lane path for levels with an even
// extent; x and y refine): vec(C) gathered from the class buffer, merged R*M
// along x, y, z into f.  Same contract as rec_load_kernel (kernels.cuh).
// ---------------------------------------------------------------------------
template <typename R, int CY, bool FAST>
__global__ void __launch_bounds__(256)
    rl2_kernel(LevelGeom<R> g, const Stencil<R> *__restrict__ stx,
               const Stencil<R> *__restrict__ sty, const Stencil<R> *__restrict__ stz,
               const R *__restrict__ cls, R *__restrict__ f, uint32_t ntx, uint32_t nty,
               uint32_t ntz) {
  using C = PairCfg<CY>;
  extern __shared__ __align__(16) unsigned char smem_bytes[];
  Carve cv{smem_bytes};
  R *V = cv.take<R>(3 * C::PLANE); // [3][BYR][64] vec(C) planes
  R *X = cv.take<R>(C::BYR * 32);  // [BYR][32]
  Stencil<R> *sY = cv.take<Stencil<R>>(CY);
  Stencil<R> *sZ = cv.take<Stencil<R>>(C::ZC);
  ClassTab *ct = cv.take<ClassTab>(1);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t nx = g.n[0], ny = g.n[1], nz = g.n[2];
  const uint32_t mx = g.m[0], my = g.m[1], mz = g.m[2];
  const bool rz = g.refine & 4;
  const uint32_t cx0 = tile_lo(blockIdx.x, ntx, mx), cx1 = tile_lo(blockIdx.x + 1, ntx, mx);
  const uint32_t cy0 = tile_lo(blockIdx.y, nty, my), cy1 = tile_lo(blockIdx.y + 1, nty, my);
  const uint32_t cz0 = tile_lo(blockIdx.z, ntz, mz), cz1 = tile_lo(blockIdx.z + 1, ntz, mz);
  const int X0 = 2 * int(cx0) - 2, Y0 = 2 * int(cy0) - 2;
  const uint32_t Z0 = rz ? (cz0 ? 2 * cz0 - 2 : 0) : cz0;
  const uint32_t Z1 = rz ? min(nz, 2 * cz1 + 1) : cz1;
  const uint64_t mxy = uint64_t(mx) * my;

  stage_stencils(sY, sty + cy0, cy1 - cy0, tid);
  if (rz)
    stage_stencils(sZ, stz + cz0, cz1 - cz0, tid);
  load_classtab(*ct, g, tid);

  const int xe = X0 + 2 * lane, xo = xe + 1;
  const bool xe_ok = xe >= 0 && xe < int(nx);
  const bool xo_ok = xo >= 0 && xo < int(nx);
  const bool xo_fine = xo_ok && xo < int(nx) - 1;
  const uint32_t cr_e = xe_ok ? uint32_t(xe) >> 1 : 0;
  const uint32_t rk_o =
      xo_fine ? uint32_t(xo - 1) >> 1 : (xo_ok ? coarse_rank(uint32_t(xo)) : 0);
  const bool xval = lane < 30 && cx0 + lane < cx1;
  const Stencil<R> sx = stx[min(cx0 + min(uint32_t(lane), 29u), mx - 1)];
  __syncthreads();

  // vec(C) plane loader: warp -> rows, lane -> pair; kept nodes read as 0
  auto load_plane = [&](uint32_t p) {
    if (p < Z1) {
      R *dst = V + (p % 3) * C::PLANE;
      const bool fz = !is_coarse(p, nz);
      const uint32_t wz = fz ? (p - 1) >> 1 : coarse_rank(p);
      for (int b = warp; b < C::BYR; b += 8) {
        const int y = Y0 + b;
        R *d = dst + b * 64 + 2 * lane;
        if (y < 0 || y >= int(ny)) {
          d[0] = R(0);
          d[1] = R(0);
          continue;
        }
        const bool fy = (y & 1) && y < int(ny) - 1;
        const uint32_t wy = fy ? (uint32_t(y) - 1) >> 1 : coarse_rank(uint32_t(y));
        const unsigned me = (unsigned(fy) << 1) | (unsigned(fz) << 2);
        const unsigned mo = me | unsigned(xo_fine);
        if (me != 0 && xe_ok)
          cp_async(d, cls + ct->row(me, wy, wz) + cr_e);
        else
          d[0] = R(0);
        if (mo != 0 && xo_ok)
          cp_async(d + 1, cls + ct->row(mo, wy, wz) + rk_o);
        else
          d[1] = R(0);
      }
    }
    cp_async_commit();
  };

  // z window c0..c3 = y results of planes p-4 .. p-1
  R c0[C::RW], c1[C::RW], c2[C::RW], c3[C::RW];
#pragma unroll
  for (int jj = 0; jj < C::RW; ++jj)
    c0[jj] = c1[jj] = c2[jj] = c3[jj] = R(0);
  const uint32_t cxo = cx0 + lane;
  load_plane(Z0);
  load_plane(Z0 + 1);
  uint32_t kk = cz0;
  for (uint32_t p = Z0; p < Z1; ++p) {
    load_plane(p + 2);
    cp_async_wait<2>();
    __syncthreads();
    const R *Vp = V + (p % 3) * C::PLANE;
    for (int b = warp; b < C::BYR; b += 8) {
      const Pair<R> v = ld_pair(Vp + b * 64 + 2 * lane);
      const R e1 = __shfl_down_sync(0xffffffffu, v.e, 1);
      const R o1 = __shfl_down_sync(0xffffffffu, v.o, 1);
      const R e2 = __shfl_down_sync(0xffffffffu, v.e, 2);
      const R xv = stencil_eval<R, FAST>(sx, v.e, v.o, e1, o1, e2);
      if (lane < 30)
        X[b * 32 + lane] = xval ? xv : R(0);
    }
    __syncthreads();
    R gv[C::RW];
#pragma unroll
    for (int jj = 0; jj < C::RW; ++jj) {
      const int j = warp + 8 * jj;
      gv[jj] = (j < CY && cy0 + j < cy1) ? y_eval<R, FAST>(sY[j], X, j, lane) : R(0);
    }
    if (!rz) {
#pragma unroll
      for (int jj = 0; jj < C::RW; ++jj) {
        const int j = warp + 8 * jj;
        if (j < CY && cy0 + j < cy1 && xval)
          f[cxo + uint64_t(mx) * (cy0 + j) + mxy * p] = gv[jj];
      }
      continue;
    }
    // emit every output whose window ends at p: centre q, d = p - q in
    // {2, 1, 0} (1 and 0 only at the last nodes, whose right taps are absent)
    while (kk < cz1) {
      const uint32_t q = coarse_pos(kk, nz);
      if (min(q + 2, nz - 1) > p)
        break;
      const Stencil<R> &s = sZ[kk - cz0];
      const uint32_t d = p - q;
#pragma unroll
      for (int jj = 0; jj < C::RW; ++jj) {
        const int j = warp + 8 * jj;
        // positions p-4 .. p are c0, c1, c2, c3, gv
        R v;
        if (d == 2)
          v = stencil_eval<R, FAST>(s, c0[jj], c1[jj], c2[jj], c3[jj], gv[jj]);
        else if (d == 1)
          v = stencil_eval<R, FAST>(s, c1[jj], c2[jj], c3[jj], gv[jj], R(0));
        else
          v = stencil_eval<R, FAST>(s, c2[jj], c3[jj], gv[jj], R(0), R(0));
        if (j < CY && cy0 + j < cy1 && xval)
          f[cxo + uint64_t(mx) * (cy0 + j) + mxy * kk] = v;
      }
      ++kk;
    }
#pragma unroll
    for (int jj = 0; jj < C::RW; ++jj) {
      c0[jj] = c1[jj];
      c1[jj] = c2[jj];
      c2[jj] = c3[jj];
      c3[jj] = gv[jj];
    }
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// Recompose GPK inverse, one level (fast path): a_l = prolongation of the
// packed coarse' values (+ class at coefficient nodes).  Lane a owns the pair
// (2(cx0+a), 2(cx0+a)+1); a warp owns output rows; the CTA marches coarse-z
// ranks, keeping the prolongated coarse planes for the fine plane between.
// cls == nullptr: classes above classes_used (read as zero).
// ---------------------------------------------------------------------------
template <typename R, int CY, bool FAST>
__global__ void __launch_bounds__(256)
    rg2_kernel(LevelGeom<R> g, const R *__restrict__ coarse, const R *__restrict__ cls,
               R *__restrict__ out, uint32_t ntx, uint32_t nty, uint32_t ntz) {
  using A = Arith<R, FAST>;
  constexpr int CR = CY + 1, CP = 33, OR = 2 * CY; // coarse rows, pitch, out rows
  extern __shared__ __align__(16) unsigned char smem_bytes[];
  Carve cv{smem_bytes};
  R *Cs = cv.take<R>(3 * CR * CP); // [3][CR][33] coarse' planes
  R *Wp = cv.take<R>(2 * OR * 64); // [2][OR][64] prolongated coarse planes
  ClassTab *ct = cv.take<ClassTab>(1);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t nx = g.n[0], ny = g.n[1], nz = g.n[2];
  const uint32_t mx = g.m[0], my = g.m[1], mz = g.m[2];
  const bool rz = g.refine & 4;
  const uint32_t cx0 = tile_lo(blockIdx.x, ntx, mx), cx1 = tile_lo(blockIdx.x + 1, ntx, mx);
  const uint32_t cy0 = tile_lo(blockIdx.y, nty, my), cy1 = tile_lo(blockIdx.y + 1, nty, my);
  const uint32_t kz0 = tile_lo(blockIdx.z, ntz, mz), kz1 = tile_lo(blockIdx.z + 1, ntz, mz);
  const uint32_t OX1 = cx1 == mx ? nx : 2 * cx1;
  const uint32_t OY1 = cy1 == my ? ny : 2 * cy1;
  const uint64_t nxy = uint64_t(nx) * ny, mxy = uint64_t(mx) * my;
  load_classtab(*ct, g, tid);

  const uint32_t xe = 2 * (cx0 + lane), xo = xe + 1;
  const bool own_e = xe < OX1, own_o = xo < OX1;
  const bool xo_fine = xo < nx - 1;
  const R tx = xo_fine ? g.r[0][xo - 1] : R(0);
  const uint32_t rk_o = xo_fine ? (xo - 1) >> 1 : coarse_rank(xo);
  // staged coarse ranks: [cx0, min(cx0+33, mx)) x [cy0, min(cy0+CR, my))
  const uint32_t ncx = min(cx0 + 33, mx) - cx0, ncy = min(cy0 + CR, my) - cy0;

  auto load_plane = [&](uint32_t k) {
    if (k < mz) {
      R *dst = Cs + (k % 3) * CR * CP;
      const R *src = coarse + mxy * k + uint64_t(cy0) * mx + cx0;
      for (uint32_t e = tid; e < ncx * ncy; e += 256) {
        const uint32_t j = e / ncx, i = e - j * ncx;
        cp_async(dst + j * CP + i, src + uint64_t(j) * mx + i);
      }
    }
    cp_async_commit();
  };

  // W of coarse row j (coarse-y rank cy0+j) at this lane's pair
  auto crow = [&](const R *Cp, int j, R &we, R &wo) {
    const R c0 = Cp[j * CP + lane];
    const R c1 = Cp[j * CP + lane + 1];
    we = c0;
    wo = xo_fine ? A::lerp(c0, c1, tx) : c1; // xo == nx-1 (even nx): coarse rank +1
  };
  auto wrow = [&](const R *Cp, uint32_t y, bool fy, R &we, R &wo) {
    if (!fy) {
      crow(Cp, int(coarse_rank(y) - cy0), we, wo);
    } else {
      const R ty = g.r[1][y - 1];
      R me_, mo_, pe_, po_;
      const int j = int((y - 1) >> 1) - int(cy0);
      crow(Cp, j, me_, mo_);
      crow(Cp, j + 1, pe_, po_);
      we = A::lerp(me_, pe_, ty);
      wo = A::lerp(mo_, po_, ty);
    }
  };

  // one output row, coalesced stores through shuffles
  auto store_row = [&](uint32_t pz, uint32_t y, R ve, R vo) {
    R *orow = out + nxy * pz + uint64_t(y) * nx + 2 * cx0;
    const int src = lane >> 1;
    const R a0 = __shfl_sync(0xffffffffu, ve, src);
    const R a1 = __shfl_sync(0xffffffffu, vo, src);
    const R b0 = __shfl_sync(0xffffffffu, ve, src + 16);
    const R b1 = __shfl_sync(0xffffffffu, vo, src + 16);
    const uint32_t x1 = 2 * cx0 + lane, x2 = x1 + 32;
    if (x1 < OX1)
      orow[lane] = (lane & 1) ? a1 : a0;
    if (x2 < OX1)
      orow[lane + 32] = (lane & 1) ? b1 : b0;
  };

  // one output plane: coarse (W from Cp, stored to wout) or fine (lerp_z)
  auto emit_plane = [&](uint32_t pz, bool fz, const R *Cp, const R *wlo, const R *whi,
                        R *wout) {
    const R tz = fz ? g.r[2][pz - 1] : R(0);
    const uint32_t wz = fz ? (pz - 1) >> 1 : coarse_rank(pz);
    for (int r = warp; r < OR; r += 8) {
      const uint32_t y = 2 * cy0 + r;
      if (y >= OY1)
        break;
      const bool fy = (y & 1) && y < ny - 1;
      R we, wo;
      if (fz) {
        const Pair<R> a = ld_pair(wlo + r * 64 + 2 * lane);
        const Pair<R> c = ld_pair(whi + r * 64 + 2 * lane);
        we = A::lerp(a.e, c.e, tz);
        wo = A::lerp(a.o, c.o, tz);
      } else {
        wrow(Cp, y, fy, we, wo);
      }
      if (wout)
        st_pair(wout + r * 64 + 2 * lane, we, wo);
      const bool fe = fy || fz, fo = fe || xo_fine;
      const uint32_t wy = fy ? (y - 1) >> 1 : coarse_rank(y);
      const unsigned me = (unsigned(fy) << 1) | (unsigned(fz) << 2);
      const unsigned mo = me | unsigned(xo_fine);
      R ve = we, vo = wo;
      if (fe) {
        const R c = (cls && own_e) ? __ldg(cls + ct->row(me, wy, wz) + (xe >> 1)) : R(0);
        ve = add(we, c);
      }
      if (fo) {
        const R c = (cls && own_o) ? __ldg(cls + ct->row(mo, wy, wz) + rk_o) : R(0);
        vo = add(wo, c);
      }
      store_row(pz, y, ve, vo);
    }
  };

  // planes of coarse ranks [kz0, kz1) plus the fine planes between k and k+1
  __syncthreads();
  load_plane(kz0);
  load_plane(kz0 + 1);
  load_plane(kz0 + 2);
  uint32_t issued = kz0 + 3;
  cp_async_wait<2>();
  __syncthreads();
  uint32_t slot = 0;
  emit_plane(rz ? coarse_pos(kz0, nz) : kz0, false, Cs + (kz0 % 3) * CR * CP, nullptr,
             nullptr, Wp);
  __syncthreads();
  for (uint32_t k = kz0; k < kz1; ++k) {
    const uint32_t p0 = rz ? coarse_pos(k, nz) : k;
    const bool has_next = k + 1 < mz;
    const uint32_t p1 = has_next ? (rz ? coarse_pos(k + 1, nz) : k + 1) : p0;
    const bool fine_between = rz && has_next && p1 == p0 + 2;
    if (!(k + 1 < kz1) && !fine_between)
      break;
    load_plane(issued++);
    cp_async_wait<2>();
    __syncthreads();
    const uint32_t ns = slot ^ 1;
    const R *Cn = Cs + ((k + 1) % 3) * CR * CP;
    if (k + 1 < kz1) {
      emit_plane(p1, false, Cn, nullptr, nullptr, rz ? Wp + ns * OR * 64 : nullptr);
    } else {
      // W of the first plane of the next chunk (needed, not emitted here)
      for (int r = warp; r < OR; r += 8) {
        const uint32_t y = 2 * cy0 + r;
        if (y >= OY1)
          break;
        R we, wo;
        wrow(Cn, y, (y & 1) && y < ny - 1, we, wo);
        st_pair(Wp + ns * OR * 64 + r * 64 + 2 * lane, we, wo);
      }
    }
    __syncthreads();
    if (fine_between)
      emit_plane(p0 + 1, true, nullptr, Wp + slot * OR * 64, Wp + ns * OR * 64, nullptr);
    __syncthreads();
    slot = ns;
  }
  cp_async_wait<0>();
}

} // namespace mgrg
