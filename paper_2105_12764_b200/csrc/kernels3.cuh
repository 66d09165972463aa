// kernels3.cuh -- lane geometry helpers of the pair-lane decompose kernel
// (kernels4.cuh): per-lane x geometry (LaneX / lane_x), class type plane
// offsets (type_plane) and the FAST 5-tap weights (W5).  The level kernel of
// this generation was superseded by kernels4.cuh and the lean family
// (lean.cuh).
#pragma once

#include "kernels2.cuh"

namespace mgrg {

template <typename R> struct LaneX {
  int xe, xo;
  bool xe_ok, xo_ok, xo_fine, own_e, own_o, xval;
  uint32_t cr_e, rk_o, otx; // coarse rank of xe, class rank of xo, x extent of xo's type
  R tx;
};

template <typename R>
__device__ __forceinline__ LaneX<R> lane_x(const LevelGeom<R> &g, int lane, uint32_t cx0,
                                          uint32_t cx1) {
  LaneX<R> L;
  const uint32_t nx = g.n[0], mx = g.m[0];
  const int X0 = 2 * int(cx0) - 2;
  const uint32_t OX1 = cx1 == mx ? nx : 2 * cx1;
  L.xe = X0 + 2 * lane;
  L.xo = L.xe + 1;
  L.xe_ok = L.xe >= 0 && L.xe < int(nx);
  L.xo_ok = L.xo >= 0 && L.xo < int(nx);
  L.xo_fine = L.xo_ok && L.xo < int(nx) - 1;
  L.own_e = lane >= 1 && L.xe < int(OX1);
  L.own_o = lane >= 1 && L.xo < int(OX1) && L.xo_ok;
  L.cr_e = L.xe_ok ? uint32_t(L.xe) >> 1 : 0;
  L.rk_o = L.xo_fine ? uint32_t(L.xo - 1) >> 1 : (L.xo_ok ? (uint32_t(L.xo) + 1) >> 1 : 0);
  L.otx = L.xo_fine ? nx - mx : mx;
  L.xval = lane < 30 && cx0 + lane < cx1;
  L.tx = L.xo_fine ? g.r[0][L.xo - 1] : R(0);
  return L;
}

// Class-type plane bases (class_slot, grid.hpp:149-164): element offset of
// (rank_x = 0, rank_y = 0, rank_z = wz) in type `mask`.
template <typename R>
__device__ __forceinline__ uint64_t type_plane(const LevelGeom<R> &g, unsigned mask,
                                               uint32_t wz) {
  return g.tbase[mask] + uint64_t(g.tex[mask]) * g.tey[mask] * wz;
}

// Five-tap weights held in registers (FAST policy).
template <typename R> struct W5 {
  R w0, w1, w2, w3, w4;
  __device__ __forceinline__ void load(const Stencil<R> &s) {
    w0 = s.w[0];
    w1 = s.w[1];
    w2 = s.w[2];
    w3 = s.w[3];
    w4 = s.w[4];
  }
  __device__ __forceinline__ R eval(R t0, R t1, R t2, R t3, R t4) const {
    R v = w0 * t0;
    v = fma(w1, t1, v);
    v = fma(w2, t2, v);
    v = fma(w3, t3, v);
    return fma(w4, t4, v);
  }
};

} // namespace mgrg
