// kernels2.cuh -- pair-per-lane level kernels (the fast path).
//
// Mapping: a warp covers one box row of 64 fine x positions; lane a owns the
// pair (X0 + 2a, X0 + 2a + 1) = (even/coarse-x node, odd/fine-x node).  With
// X0 = 2*cx0 - 2 the 32 pairs cover the reach-2 stencil window of 30 coarse-x
// outputs, so the merged R*M along x is a 5-tap window over lanes i, i+1,
// i+2 and runs on warp shuffles with the lane's stencil coefficients held in
// registers.  No integer division, no per-node type switch.
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
#pragma once

#include "common.cuh"
#include "level.cuh"

namespace mgrg {

// One coarse output of the merged mass-trans along a dimension, as host-
// precomputed coefficients in the working precision (see stencil.hpp).
// v = mv(q) [+ cl*mv(q-1)] [+ cr*mv(q+1)]   (masstrans_window,
// kernels.hpp:159-178), taps in(q-2..q+2).
template <typename R> struct Stencil {
  R hm2, hm1, h0, hp1; // h[q-2], h[q-1], h[q], h[q+1]
  R dm1, d0, dp1;      // 2(h[j-1]+h[j]) at j = q-1, q, q+1 (boundary: 2h)
  R cl, cr;            // r[q-2], 1 - r[q]
  uint32_t flags;      // ST_* below
};
enum : uint32_t {
  ST_LEFT = 1,   // q == 0: mv(q) = 2h0*in(q) + h0*in(q+1)
  ST_RIGHT = 2,  // q == n-1: mv(q) = h[n-2]*in(q-1) + 2h[n-2]*in(q)
  ST_HASL = 4,   // q-1 is fine: + r[q-2]*mv(q-1)
  ST_HASR = 8,   // q+1 is fine: + (1-r[q])*mv(q+1)
  ST_SHIFT = 16, // q = 2c-1 (last node of an even extent): taps shifted by one
  ST_VALID = 32
};

// Taps t0..t4 are the fine positions 2c-2 .. 2c+2 relative to the output's
// nominal centre 2c; ST_SHIFT moves the centre to 2c-1.
template <typename R>
__device__ __forceinline__ R stencil_eval(const Stencil<R> &s, R t0, R t1, R t2, R t3,
                                          R t4) {
  if (s.flags & ST_SHIFT) { // q = 2c-1 = n-1, n even: only the right-boundary mv
    return add(mul(s.hm1, t0), mul(s.d0, t1));
  }
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

template <typename R>
__device__ __forceinline__ Stencil<R> load_stencil(const Stencil<R> *p) {
  Stencil<R> s;
  s.hm2 = __ldg(&p->hm2);
  s.hm1 = __ldg(&p->hm1);
  s.h0 = __ldg(&p->h0);
  s.hp1 = __ldg(&p->hp1);
  s.dm1 = __ldg(&p->dm1);
  s.d0 = __ldg(&p->d0);
  s.dp1 = __ldg(&p->dp1);
  s.cl = __ldg(&p->cl);
  s.cr = __ldg(&p->cr);
  s.flags = __ldg(&p->flags);
  return s;
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

// Geometry common to the three pair-lane kernels.
struct TileGeo {
  uint32_t cx0, cx1, cy0, cy1;
  int X0, Y0;               // fine box origin (may be negative)
  uint32_t OX1, OY0, OY1;   // ownership (x starts at 2*cx0)
};

template <int CY> struct PairCfg {
  static constexpr int NW = 8, T = 256, BX = 64, BYR = 2 * CY + 3;
  static constexpr int PLANE = BYR * BX;
};

template <typename R, int CY> constexpr size_t dec2_smem() {
  using C = PairCfg<CY>;
  return sizeof(R) * (4 * C::PLANE + 2 * C::PLANE + C::BYR * 32 + 5 * CY * 32);
}
template <typename R, int CY> constexpr size_t rl2_smem() {
  using C = PairCfg<CY>;
  return sizeof(R) * (3 * C::PLANE + C::BYR * 32 + 5 * CY * 32);
}
template <typename R, int CY> constexpr size_t rg2_smem() {
  // coarse planes: 3 x (CY+1) rows x 33 (padded to 16 B); W planes: 2 x 2CY x 64
  return sizeof(R) * (((3 * (CY + 1) * 33 + 3) & ~3) + 2 * (2 * CY) * 64);
}

// y pass of one plane p for this warp's output rows j (CY/8 of them): the
// result goes to f directly when z does not refine, else into the z ring G.
template <typename R, int CY>
__device__ __forceinline__ void y_stage(const LevelGeom<R> &g, const Stencil<R> *sty,
                                        const R *X, R *G, const TileGeo &tg, int warp,
                                        int lane, uint32_t p, R *__restrict__ f) {
  const uint32_t mx = g.m[0], my = g.m[1];
  const uint32_t cx = tg.cx0 + lane;
  const bool xval = lane < 30 && cx < tg.cx1;
#pragma unroll
  for (int jj = 0; jj < (CY + 7) / 8; ++jj) {
    const int j = warp + 8 * jj;
    const uint32_t cy = tg.cy0 + j;
    if (j < CY && cy < tg.cy1) {
      const Stencil<R> s = load_stencil(sty + cy);
      const R *c = X + (2 * j) * 32 + lane; // box rows 2j .. 2j+4
      const R v = stencil_eval(s, c[0], c[32], c[64], c[96], c[128]);
      if (!(g.refine & 4)) {
        if (xval)
          f[cx + uint64_t(mx) * (cy + uint64_t(my) * p)] = v;
      } else {
        G[((p % 5) * CY + j) * 32 + lane] = v;
      }
    }
  }
}

// z stage: emit every coarse-z output whose 5-plane window is complete
// (all positions <= `processed` are in the ring).  G is indexed by position,
// so z descriptors are built unshifted.
template <typename R, int CY>
__device__ __forceinline__ void z_stage(const LevelGeom<R> &g, const Stencil<R> *stz,
                                        const R *G, const TileGeo &tg, int warp, int lane,
                                        R *__restrict__ f, uint32_t cz1, uint32_t &kk,
                                        uint32_t processed) {
  const uint32_t mx = g.m[0], my = g.m[1], nz = g.n[2];
  const uint64_t mxy = uint64_t(mx) * my;
  const uint32_t cx = tg.cx0 + lane;
  const bool xval = lane < 30 && cx < tg.cx1;
  while (kk < cz1) {
    const uint32_t q = coarse_pos(kk, nz);
    if (min(q + 2, nz - 1) > processed)
      break;
    const Stencil<R> s = load_stencil(stz + kk);
#pragma unroll
    for (int jj = 0; jj < (CY + 7) / 8; ++jj) {
      const int j = warp + 8 * jj;
      const uint32_t cy = tg.cy0 + j;
      if (j < CY && cy < tg.cy1 && xval) {
        auto gv = [&](int pos) -> R {
          return (pos < 0 || pos >= int(nz)) ? R(0) : G[((pos % 5) * CY + j) * 32 + lane];
        };
        const int qi = int(q);
        const R v = stencil_eval(s, gv(qi - 2), gv(qi - 1), gv(qi), gv(qi + 1), gv(qi + 2));
        f[cx + uint64_t(mx) * cy + mxy * kk] = v;
      }
    }
    ++kk;
  }
}

// ---------------------------------------------------------------------------
// Decompose, one level (fast path; x and y refine).  Same contract as
// dec_level_kernel (kernels.cuh).
// ---------------------------------------------------------------------------
template <typename R, int CY>
__global__ void __launch_bounds__(256)
    dec2_kernel(LevelGeom<R> g, const Stencil<R> *__restrict__ stx,
                const Stencil<R> *__restrict__ sty, const Stencil<R> *__restrict__ stz,
                const R *__restrict__ in, R *__restrict__ cls, R *__restrict__ P,
                R *__restrict__ f, uint32_t ntx, uint32_t nty, uint32_t ntz) {
  using C = PairCfg<CY>;
  extern __shared__ __align__(16) unsigned char smem_bytes[];
  R *U = reinterpret_cast<R *>(smem_bytes); // [4][BYR][64] raw planes
  R *Wc = U + 4 * C::PLANE;                 // [2][BYR][64] prolongated coarse planes
  R *X = Wc + 2 * C::PLANE;                 // [BYR][32] x-pass results
  R *G = X + C::BYR * 32;                   // [5][CY][32] xy results (z ring)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t nx = g.n[0], ny = g.n[1], nz = g.n[2];
  const uint32_t mx = g.m[0], my = g.m[1], mz = g.m[2];
  const bool rz = g.refine & 4;
  TileGeo tg;
  tg.cx0 = tile_lo(blockIdx.x, ntx, mx);
  tg.cx1 = tile_lo(blockIdx.x + 1, ntx, mx);
  tg.cy0 = tile_lo(blockIdx.y, nty, my);
  tg.cy1 = tile_lo(blockIdx.y + 1, nty, my);
  const uint32_t cz0 = tile_lo(blockIdx.z, ntz, mz), cz1 = tile_lo(blockIdx.z + 1, ntz, mz);
  tg.X0 = 2 * int(tg.cx0) - 2;
  tg.Y0 = 2 * int(tg.cy0) - 2;
  tg.OX1 = tg.cx1 == mx ? nx : 2 * tg.cx1;
  tg.OY0 = 2 * tg.cy0;
  tg.OY1 = tg.cy1 == my ? ny : 2 * tg.cy1;
  const uint32_t Z0 = rz ? (cz0 ? 2 * cz0 - 2 : 0) : cz0;
  const uint32_t Z1 = rz ? min(nz, 2 * cz1 + 1) : cz1;
  const uint32_t OZ0 = rz ? 2 * cz0 : cz0, OZ1 = rz ? (cz1 == mz ? nz : 2 * cz1) : cz1;
  const uint64_t nxy = uint64_t(nx) * ny;

  // ---- per-lane x geometry
  const int xe = tg.X0 + 2 * lane, xo = xe + 1;
  const bool xo_ok = xo >= 0 && xo < int(nx);
  const bool xo_fine = xo_ok && xo < int(nx) - 1;
  const R tx = xo_fine ? __ldg(g.r[0] + xo - 1) : R(0);
  const bool own_e = lane >= 1 && xe < int(tg.OX1);
  const bool own_o = lane >= 1 && xo < int(tg.OX1) && xo_ok;
  const uint32_t cr_e = uint32_t(xe) >> 1;                         // coarse rank of xe
  const uint32_t rk_o = xo_fine ? uint32_t(xo - 1) >> 1 : coarse_rank(uint32_t(xo));
  Stencil<R> sx{};
  const bool xval = lane < 30 && tg.cx0 + lane < tg.cx1;
  if (xval)
    sx = load_stencil(stx + tg.cx0 + lane);

  // ---- LDGSTS plane loader: thread -> column tid&63, rows (tid>>6) + 4m
  const int lc = tid & 63, lr0 = tid >> 6;
  const int gx = tg.X0 + lc;
  const bool col_ok = gx >= 0 && gx < int(nx);
  auto load_plane = [&](uint32_t p) {
    if (p < Z1 && col_ok) {
      R *dst = U + (p & 3) * C::PLANE + lc;
      const R *src = in + nxy * p + gx;
#pragma unroll 4
      for (int b = lr0; b < C::BYR; b += 4) {
        const int gy = tg.Y0 + b;
        if (gy >= 0 && gy < int(ny))
          cp_async(dst + b * 64, src + uint64_t(gy) * nx);
      }
    }
    cp_async_commit();
  };

  // ---- GPK + stores + x pass for one plane.  Fine plane: wlo/whi are the
  // prolongated neighbour coarse planes.  Coarse plane: wout receives W.
  auto process_plane = [&](uint32_t p, bool fz, const R *wlo, const R *whi, R *wout) {
    const R *Up = U + (p & 3) * C::PLANE;
    const R tz = fz ? __ldg(g.r[2] + p - 1) : R(0);
    const bool ownz = p >= OZ0 && p < OZ1;
    const uint32_t wz = fz ? (p - 1) >> 1 : coarse_rank(p);
    for (int b = warp; b < C::BYR; b += 8) {
      const int y = tg.Y0 + b;
      const bool y_ok = y >= 0 && y < int(ny);
      const bool fy = y_ok && (y & 1) && y < int(ny) - 1;
      const Pair<R> u = ld_pair(Up + b * 64 + 2 * lane);
      R we, wo;
      if (fz) {
        const Pair<R> a = ld_pair(wlo + b * 64 + 2 * lane);
        const Pair<R> c = ld_pair(whi + b * 64 + 2 * lane);
        we = lerp(a.e, c.e, tz);
        wo = lerp(a.o, c.o, tz);
      } else if (!fy) {
        const R un = __shfl_down_sync(0xffffffffu, u.e, 1);
        we = u.e;
        wo = xo_fine ? lerp(u.e, un, tx) : u.o;
      } else {
        const R ty = __ldg(g.r[1] + y - 1);
        const Pair<R> um = ld_pair(Up + (b - 1) * 64 + 2 * lane);
        const Pair<R> up = ld_pair(Up + (b + 1) * 64 + 2 * lane);
        const R umn = __shfl_down_sync(0xffffffffu, um.e, 1);
        const R upn = __shfl_down_sync(0xffffffffu, up.e, 1);
        const R wmo = xo_fine ? lerp(um.e, umn, tx) : um.o;
        const R wpo = xo_fine ? lerp(up.e, upn, tx) : up.o;
        we = lerp(um.e, up.e, ty);
        wo = lerp(wmo, wpo, ty);
      }
      if (wout)
        st_pair(wout + b * 64 + 2 * lane, we, wo);
      const bool fe = fy || fz;          // even-x node is a coefficient node
      const bool fo = fe || xo_fine;     // odd-x node is a coefficient node
      const R ve = fe ? sub(u.e, we) : R(0);
      const R vo = fo ? sub(u.o, wo) : R(0);
      // class order / packed-coarse stores of owned nodes (coalesced runs)
      if (ownz && y_ok && uint32_t(y) >= tg.OY0 && uint32_t(y) < tg.OY1) {
        const uint32_t wy = fy ? (uint32_t(y) - 1) >> 1 : coarse_rank(uint32_t(y));
        const unsigned me = (unsigned(fy) << 1) | (unsigned(fz) << 2);
        if (own_e) {
          if (me == 0)
            P[cr_e + uint64_t(mx) * (wy + uint64_t(my) * wz)] = u.e;
          else
            cls[g.tbase[me] + cr_e + uint64_t(g.tex[me]) * (wy + uint64_t(g.tey[me]) * wz)] = ve;
        }
        if (own_o) {
          const unsigned mo = me | unsigned(xo_fine);
          if (mo == 0)
            P[rk_o + uint64_t(mx) * (wy + uint64_t(my) * wz)] = u.o;
          else
            cls[g.tbase[mo] + rk_o + uint64_t(g.tex[mo]) * (wy + uint64_t(g.tey[mo]) * wz)] = vo;
        }
      }
      // x pass: output lane i from pairs i, i+1 and the even node of i+2
      const R e1 = __shfl_down_sync(0xffffffffu, ve, 1);
      const R o1 = __shfl_down_sync(0xffffffffu, vo, 1);
      const R e2 = __shfl_down_sync(0xffffffffu, ve, 2);
      if (lane < 30)
        X[b * 32 + lane] = xval ? stencil_eval(sx, ve, vo, e1, o1, e2) : R(0);
    }
  };

  uint32_t kk = cz0;
  // prologue: three planes in flight
  load_plane(Z0);
  load_plane(Z0 + 1);
  load_plane(Z0 + 2);
  uint32_t issued = Z0 + 3;
  cp_async_wait<2>();
  __syncthreads();
  if (!rz) {
    // z does not refine: every plane is coarse and is its own output
    for (uint32_t p = Z0; p < Z1; ++p) {
      if (p > Z0) {
        load_plane(issued++);
        cp_async_wait<2>();
        __syncthreads();
      }
      process_plane(p, false, nullptr, nullptr, nullptr);
      __syncthreads();
      y_stage<R, CY>(g, sty, X, G, tg, warp, lane, p, f);
      __syncthreads();
    }
    cp_async_wait<0>();
    return;
  }
  uint32_t pc = Z0; // last processed coarse plane
  uint32_t slot = 0;
  process_plane(pc, false, nullptr, nullptr, Wc);
  __syncthreads();
  y_stage<R, CY>(g, sty, X, G, tg, warp, lane, pc, f);
  __syncthreads();
  for (;;) {
    const uint32_t nxt = pc + 2 <= nz - 1 ? pc + 2 : pc + 1;
    if (nxt >= Z1)
      break;
    load_plane(issued++);
    load_plane(issued++);
    cp_async_wait<2>();
    __syncthreads();
    const uint32_t ns = slot ^ 1;
    process_plane(nxt, false, nullptr, nullptr, Wc + ns * C::PLANE);
    __syncthreads();
    y_stage<R, CY>(g, sty, X, G, tg, warp, lane, nxt, f);
    __syncthreads();
    if (nxt == pc + 2) { // the fine plane between the two coarse planes
      process_plane(pc + 1, true, Wc + slot * C::PLANE, Wc + ns * C::PLANE, nullptr);
      __syncthreads();
      y_stage<R, CY>(g, sty, X, G, tg, warp, lane, pc + 1, f);
    }
    z_stage<R, CY>(g, stz, G, tg, warp, lane, f, cz1, kk, nxt);
    __syncthreads();
    pc = nxt;
    slot = ns;
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// Recompose load vector, one level (fast path): vec(C) gathered from class l
// in coalesced per-row runs (lane a reads the a-th coarse-x and the a-th
// fine-x entry of the row's two class types) into a 3-plane ring, then the
// same x (shuffle) / y / z merged mass-trans as dec2.
// ---------------------------------------------------------------------------
template <typename R, int CY>
__global__ void __launch_bounds__(256)
    rl2_kernel(LevelGeom<R> g, const Stencil<R> *__restrict__ stx,
               const Stencil<R> *__restrict__ sty, const Stencil<R> *__restrict__ stz,
               const R *__restrict__ cls, R *__restrict__ f, uint32_t ntx, uint32_t nty,
               uint32_t ntz) {
  using C = PairCfg<CY>;
  extern __shared__ __align__(16) unsigned char smem_bytes[];
  R *V = reinterpret_cast<R *>(smem_bytes); // [3][BYR][64] vec(C) planes
  R *X = V + 3 * C::PLANE;                  // [BYR][32]
  R *G = X + C::BYR * 32;                   // [5][CY][32]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t nx = g.n[0], ny = g.n[1], nz = g.n[2];
  const uint32_t mx = g.m[0], my = g.m[1], mz = g.m[2];
  const bool rz = g.refine & 4;
  TileGeo tg;
  tg.cx0 = tile_lo(blockIdx.x, ntx, mx);
  tg.cx1 = tile_lo(blockIdx.x + 1, ntx, mx);
  tg.cy0 = tile_lo(blockIdx.y, nty, my);
  tg.cy1 = tile_lo(blockIdx.y + 1, nty, my);
  const uint32_t cz0 = tile_lo(blockIdx.z, ntz, mz), cz1 = tile_lo(blockIdx.z + 1, ntz, mz);
  tg.X0 = 2 * int(tg.cx0) - 2;
  tg.Y0 = 2 * int(tg.cy0) - 2;
  const uint32_t Z0 = rz ? (cz0 ? 2 * cz0 - 2 : 0) : cz0;
  const uint32_t Z1 = rz ? min(nz, 2 * cz1 + 1) : cz1;

  const int xe = tg.X0 + 2 * lane, xo = xe + 1;
  const bool xe_ok = xe >= 0 && xe < int(nx);
  const bool xo_ok = xo >= 0 && xo < int(nx);
  const bool xo_fine = xo_ok && xo < int(nx) - 1;
  const uint32_t cr_e = xe_ok ? uint32_t(xe) >> 1 : 0;
  const uint32_t rk_o = xo_fine ? uint32_t(xo - 1) >> 1 : 0;
  Stencil<R> sx{};
  const bool xval = lane < 30 && tg.cx0 + lane < tg.cx1;
  if (xval)
    sx = load_stencil(stx + tg.cx0 + lane);

  // vec(C) plane loader: warp -> rows, lane -> pair; coarse nodes read as 0
  auto load_plane = [&](uint32_t p) {
    if (p < Z1) {
      R *dst = V + (p % 3) * C::PLANE;
      const bool fz = !is_coarse(p, nz);
      const uint32_t wz = fz ? (p - 1) >> 1 : coarse_rank(p);
      for (int b = warp; b < C::BYR; b += 8) {
        const int y = tg.Y0 + b;
        R *d = dst + b * 64 + 2 * lane;
        if (y < 0 || y >= int(ny)) {
          d[0] = R(0);
          d[1] = R(0);
          continue;
        }
        const bool fy = (y & 1) && y < int(ny) - 1;
        const uint32_t wy = fy ? (uint32_t(y) - 1) >> 1 : coarse_rank(uint32_t(y));
        const unsigned me = (unsigned(fy) << 1) | (unsigned(fz) << 2);
        if (me != 0 && xe_ok)
          cp_async(d, cls + g.tbase[me] + cr_e +
                          uint64_t(g.tex[me]) * (wy + uint64_t(g.tey[me]) * wz));
        else
          d[0] = R(0);
        const unsigned mo = me | 1u;
        if (xo_fine)
          cp_async(d + 1, cls + g.tbase[mo] + rk_o +
                              uint64_t(g.tex[mo]) * (wy + uint64_t(g.tey[mo]) * wz));
        else if (xo_ok && me != 0) // last node of an even extent: coarse in x
          cp_async(d + 1, cls + g.tbase[me] + coarse_rank(uint32_t(xo)) +
                              uint64_t(g.tex[me]) * (wy + uint64_t(g.tey[me]) * wz));
        else
          d[1] = R(0);
      }
    }
    cp_async_commit();
  };

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
      if (lane < 30)
        X[b * 32 + lane] = xval ? stencil_eval(sx, v.e, v.o, e1, o1, e2) : R(0);
    }
    __syncthreads();
    y_stage<R, CY>(g, sty, X, G, tg, warp, lane, p, f);
    if (rz)
      z_stage<R, CY>(g, stz, G, tg, warp, lane, f, cz1, kk, p);
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
template <typename R, int CY>
__global__ void __launch_bounds__(256)
    rg2_kernel(LevelGeom<R> g, const R *__restrict__ coarse, const R *__restrict__ cls,
               R *__restrict__ out, uint32_t ntx, uint32_t nty, uint32_t ntz) {
  constexpr int CR = CY + 1, CP = 33, OR = 2 * CY; // coarse rows, pitch, out rows
  extern __shared__ __align__(16) unsigned char smem_bytes[];
  R *Cs = reinterpret_cast<R *>(smem_bytes); // [3][CR][33] coarse' planes
  R *Wp = Cs + ((3 * CR * CP + 3) & ~3);     // [2][OR][64] prolongated coarse planes

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

  const uint32_t xe = 2 * (cx0 + lane), xo = xe + 1;
  const bool own_e = xe < OX1, own_o = xo < OX1;
  const bool xo_fine = xo < nx - 1;
  const R tx = xo_fine ? __ldg(g.r[0] + xo - 1) : R(0);
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

  // value of coarse row j (coarse-y rank cy0+j) of plane C at this lane's pair
  auto crow = [&](const R *Cp, int j, R &we, R &wo) {
    const R c0 = Cp[j * CP + lane];
    const R c1 = Cp[j * CP + lane + 1];
    we = c0;
    wo = xo_fine ? lerp(c0, c1, tx) : c1; // xo == nx-1 (even nx): coarse rank +1
  };

  // writes one output row (fine y), with coalesced stores through shuffles
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
    const R tz = fz ? __ldg(g.r[2] + pz - 1) : R(0);
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
        we = lerp(a.e, c.e, tz);
        wo = lerp(a.o, c.o, tz);
      } else if (!fy) {
        crow(Cp, int(coarse_rank(y) - cy0), we, wo);
      } else {
        const R ty = __ldg(g.r[1] + y - 1);
        R me_, mo_, pe_, po_;
        const int j = int((y - 1) >> 1) - int(cy0);
        crow(Cp, j, me_, mo_);
        crow(Cp, j + 1, pe_, po_);
        we = lerp(me_, pe_, ty);
        wo = lerp(mo_, po_, ty);
      }
      if (wout)
        st_pair(wout + r * 64 + 2 * lane, we, wo);
      const bool fe = fy || fz, fo = fe || xo_fine;
      const uint32_t wy = fy ? (y - 1) >> 1 : coarse_rank(y);
      const unsigned me = (unsigned(fy) << 1) | (unsigned(fz) << 2);
      R ve = we, vo = wo;
      if (fe) {
        const R c = (cls && own_e)
                        ? __ldg(cls + g.tbase[me] + (xe >> 1) +
                                uint64_t(g.tex[me]) * (wy + uint64_t(g.tey[me]) * wz))
                        : R(0);
        ve = add(we, c);
      }
      if (fo) {
        const unsigned mo = me | unsigned(xo_fine);
        const uint32_t rx = xo_fine ? (xo - 1) >> 1 : coarse_rank(xo);
        const R c = (cls && own_o)
                        ? __ldg(cls + g.tbase[mo] + rx +
                                uint64_t(g.tex[mo]) * (wy + uint64_t(g.tey[mo]) * wz))
                        : R(0);
        vo = add(wo, c);
      }
      store_row(pz, y, ve, vo);
    }
  };

  // planes of coarse ranks [kz0, kz1) plus the fine planes between k and k+1
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
    // coarse plane k+1: emitted only inside the chunk, prolongated W needed
    // by the fine plane between k and k+1 either way
    if (k + 1 < kz1)
      emit_plane(p1, false, Cs + ((k + 1) % 3) * CR * CP, nullptr, nullptr,
                 rz ? Wp + ns * OR * 64 : nullptr);
    else if (fine_between) {
      // W of the first plane of the next chunk (not emitted here)
      const R *Cp = Cs + ((k + 1) % 3) * CR * CP;
      for (int r = warp; r < OR; r += 8) {
        const uint32_t y = 2 * cy0 + r;
        if (y >= OY1)
          break;
        const bool fy = (y & 1) && y < ny - 1;
        R we, wo;
        if (!fy) {
          crow(Cp, int(coarse_rank(y) - cy0), we, wo);
        } else {
          const R ty = __ldg(g.r[1] + y - 1);
          R me_, mo_, pe_, po_;
          const int j = int((y - 1) >> 1) - int(cy0);
          crow(Cp, j, me_, mo_);
          crow(Cp, j + 1, pe_, po_);
          we = lerp(me_, pe_, ty);
          wo = lerp(mo_, po_, ty);
        }
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
