// kernels3.cuh -- lean pair-lane level kernels (x and y refine).
//
// Same decomposition of the work as kernels2.cuh (a warp row covers 64 fine
// x positions, lane a owns the pair (X0 + 2a, X0 + 2a + 1); x pass on warp
// shuffles, y pass through shared memory, z pass in registers; GPK as
// prolongation x -> y -> z, bit-identical to interpolate_node), rewritten
// for instruction count -- the ncu capture of the kernels2 version showed
// them issue-bound (78 % issue-active, 4.7 warp instructions per fine
// element at 1025^3) while DRAM ran at 20 %:
//   * per-row class / packed-coarse offsets are computed once per CTA
//     (plane independent: offset = extent_x(mask) * rank_y + rank_x) and per
//     plane only four base pointers change;
//   * warp-uniform row kinds (warps own rows b = warp + 8i, all of one
//     parity) select straight-line code; kept-node rows skip the even-tap
//     shuffles and multiplies;
//   * the LDGSTS staging advances precomputed pointers with a per-thread
//     row-validity mask instead of recomputing 64-bit addresses per element;
//   * the FAST policy keeps the y-stencil weights in registers.
#pragma once

#include "kernels2.cuh"

namespace mgrg {

template <typename R> constexpr int cy3() { return sizeof(R) == 4 ? 16 : 8; }

template <int CY> struct T3 {
  static constexpr int NW = 8, T = 256;
  static constexpr int BYR = 2 * CY + 3;         // box rows
  static constexpr int NI = (BYR + NW - 1) / NW; // rows per warp
  static constexpr int RW = (CY + NW - 1) / NW;  // y outputs per warp
  static constexpr int PL = BYR * 64;            // plane elements
  static constexpr int ZC = 32;                  // coarse-z outputs per CTA
  static constexpr int NQ = (BYR + 3) / 4;       // staging rows per thread
};

template <typename R, int CY> constexpr size_t dec3_smem() {
  using C = T3<CY>;
  return al16(sizeof(R) * 6 * C::PL) + al16(sizeof(R) * C::BYR * 32) +
         al16(sizeof(Stencil<R>) * CY) + al16(sizeof(Stencil<R>) * C::ZC) +
         al16(sizeof(R) * (2 * C::ZC + 4));
}

// Per-CTA x geometry of this lane (registers for the whole kernel).
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

// ---------------------------------------------------------------------------
// Decompose, one level: GPK forward on `in`, class-order store into `cls`,
// packed kept-node values into P, merged R*M of vec(C) into f
// (refactor.hpp:165-175 minus the solves; kernels.hpp:231-279, 158-185).
// ---------------------------------------------------------------------------
template <typename R, int CY, bool FAST, int MINB = 3>
__global__ void __launch_bounds__(256, MINB)
    dec3_kernel(LevelGeom<R> g, const Stencil<R> *__restrict__ stx,
                const Stencil<R> *__restrict__ sty, const Stencil<R> *__restrict__ stz,
                const R *__restrict__ in, R *__restrict__ cls, R *__restrict__ P,
                R *__restrict__ f, uint32_t ntx, uint32_t nty, uint32_t ntz) {
  using C = T3<CY>;
  using A = Arith<R, FAST>;
  extern __shared__ __align__(16) unsigned char smem_bytes[];
  Carve cv{smem_bytes};
  R *U = cv.take<R>(6 * C::PL); // [4][BYR][64] raw planes + [2][BYR][64] W planes
  R *Wc = U + 4 * C::PL;
  R *X = cv.take<R>(C::BYR * 32); // [BYR][32] x-pass results
  Stencil<R> *sY = cv.take<Stencil<R>>(CY);
  Stencil<R> *sZ = cv.take<Stencil<R>>(C::ZC);
  R *tzv = cv.take<R>(2 * C::ZC + 4); // r_z of each box plane (fine planes)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t nx = g.n[0], ny = g.n[1], nz = g.n[2];
  const uint32_t mx = g.m[0], my = g.m[1], mz = g.m[2];
  const bool rz = g.refine & 4;
  const uint32_t cx0 = tile_lo(blockIdx.x, ntx, mx), cx1 = tile_lo(blockIdx.x + 1, ntx, mx);
  const uint32_t cy0 = tile_lo(blockIdx.y, nty, my), cy1 = tile_lo(blockIdx.y + 1, nty, my);
  const uint32_t cz0 = tile_lo(blockIdx.z, ntz, mz), cz1 = tile_lo(blockIdx.z + 1, ntz, mz);
  const int X0 = 2 * int(cx0) - 2, Y0 = 2 * int(cy0) - 2;
  const uint32_t OY0 = 2 * cy0, OY1 = cy1 == my ? ny : 2 * cy1;
  const uint32_t Z0 = rz ? (cz0 ? 2 * cz0 - 2 : 0) : cz0;
  const uint32_t Z1 = rz ? min(nz, 2 * cz1 + 1) : cz1;
  const uint32_t OZ0 = rz ? 2 * cz0 : cz0, OZ1 = rz ? (cz1 == mz ? nz : 2 * cz1) : cz1;
  const uint64_t nxy = uint64_t(nx) * ny;
  const uint64_t mxy = uint64_t(mx) * my;

  // ---- per-CTA tables
  stage_stencils(sY, sty + cy0, cy1 - cy0, tid);
  if (rz) {
    stage_stencils(sZ, stz + cz0, cz1 - cz0, tid);
    for (uint32_t p = Z0 + tid; p < Z1; p += 256)
      tzv[p - Z0] = ((p & 1) && p < nz - 1) ? g.r[2][p - 1] : R(0);
  }

  // ---- per-lane x geometry and x stencil (registers)
  const LaneX<R> lx = lane_x(g, lane, cx0, cx1);
  const Stencil<R> sx = stx[min(cx0 + min(uint32_t(lane), 29u), mx - 1)];
  W5<R> wx;
  if constexpr (FAST)
    wx.load(sx);

  // ---- per-row constants (plane independent): rows b = warp + 8i
  uint32_t rowE[C::NI], rowO[C::NI];
  R tyr[C::NI];
  uint32_t yok = 0, fyb = 0, owny = 0;
#pragma unroll
  for (int i = 0; i < C::NI; ++i) {
    const int b = warp + 8 * i;
    const int y = Y0 + b;
    const bool ok = b < C::BYR && y >= 0 && y < int(ny);
    const bool fy = ok && (y & 1) && y < int(ny) - 1;
    const uint32_t wy = ok ? (fy ? uint32_t(y) >> 1 : (uint32_t(y) + 1) >> 1) : 0;
    rowE[i] = mx * wy + lx.cr_e;
    rowO[i] = lx.otx * wy + lx.rk_o;
    tyr[i] = fy ? g.r[1][y - 1] : R(0);
    yok |= uint32_t(ok) << i;
    fyb |= uint32_t(fy) << i;
    owny |= uint32_t(ok && uint32_t(y) >= OY0 && uint32_t(y) < OY1) << i;
  }

  // ---- LDGSTS staging: thread -> column tid & 63, rows (tid >> 6) + 4q
  const int lc = tid & 63, lr0 = tid >> 6;
  const int gx = X0 + lc;
  uint32_t ldmask = 0;
#pragma unroll
  for (int q = 0; q < C::NQ; ++q) {
    const int b = lr0 + 4 * q, gy = Y0 + b;
    ldmask |= uint32_t(b < C::BYR && gy >= 0 && gy < int(ny)) << q;
  }
  if (!(gx >= 0 && gx < int(nx)))
    ldmask = 0;
  const R *ldbase = in + gx + int64_t(Y0 + lr0) * int64_t(nx);
  auto load_plane = [&](uint32_t p) {
    if (p < Z1) {
      R *dst = U + (p & 3) * C::PL + lr0 * 64 + lc;
      const R *src = ldbase + nxy * p;
#pragma unroll
      for (int q = 0; q < C::NQ; ++q)
        if ((ldmask >> q) & 1)
          cp_async(dst + q * 4 * 64, src + int64_t(q) * 4 * nx);
    }
    cp_async_commit();
  };

  // ---- one plane: GPK + stores + x pass.  Fine plane: wlo/whi are the
  // neighbouring coarse planes' W.  Coarse plane: W goes to wout.
  auto process_plane = [&](uint32_t p, bool fz, const R *wlo, const R *whi, R *wout) {
    const R *Up = U + (p & 3) * C::PL;
    const R tz = fz ? tzv[p - Z0] : R(0);
    const bool ownz = p >= OZ0 && p < OZ1;
    const uint32_t wz = fz ? p >> 1 : (p + 1) >> 1;
    // plane bases of the row kinds (coarse row / fine row) for the even and
    // odd node of the pair; kept nodes go to P
    const unsigned mz_ = fz ? 4u : 0u;
    R *eB0 = fz ? cls + type_plane(g, mz_, wz) : P + mxy * wz;
    R *eB1 = cls + type_plane(g, mz_ | 2u, wz);
    R *oB0 = lx.xo_fine ? cls + type_plane(g, mz_ | 1u, wz) : eB0;
    R *oB1 = lx.xo_fine ? cls + type_plane(g, mz_ | 3u, wz) : eB1;
#pragma unroll
    for (int i = 0; i < C::NI; ++i) {
      const int b = warp + 8 * i;
      if (b >= C::BYR)
        break;
      const bool ok = (yok >> i) & 1, fy = (fyb >> i) & 1;
      R ve = R(0), vo = R(0);
      if (ok) {
        const Pair<R> u = ld_pair(Up + b * 64 + 2 * lane);
        R we, wo;
        const bool kept_row = !fz && !fy; // coarse row of a coarse plane
        if (fz) {
          const Pair<R> a = ld_pair(wlo + b * 64 + 2 * lane);
          const Pair<R> c = ld_pair(whi + b * 64 + 2 * lane);
          we = A::lerp(a.e, c.e, tz);
          wo = A::lerp(a.o, c.o, tz);
        } else if (!fy) {
          const R un = __shfl_down_sync(0xffffffffu, u.e, 1);
          we = u.e;
          wo = lx.xo_fine ? A::lerp(u.e, un, lx.tx) : u.o;
        } else {
          const Pair<R> um = ld_pair(Up + (b - 1) * 64 + 2 * lane);
          const Pair<R> up = ld_pair(Up + (b + 1) * 64 + 2 * lane);
          const R umn = __shfl_down_sync(0xffffffffu, um.e, 1);
          const R upn = __shfl_down_sync(0xffffffffu, up.e, 1);
          const R wmo = lx.xo_fine ? A::lerp(um.e, umn, lx.tx) : um.o;
          const R wpo = lx.xo_fine ? A::lerp(up.e, upn, lx.tx) : up.o;
          we = A::lerp(um.e, up.e, tyr[i]);
          wo = A::lerp(wmo, wpo, tyr[i]);
        }
        if (wout)
          st_pair(wout + b * 64 + 2 * lane, we, wo);
        // vec(C): coefficients at coefficient nodes, 0 at kept nodes and
        // outside the grid
        if (!kept_row && lx.xe_ok)
          ve = sub(u.e, we);
        if (lx.xo_ok && (lx.xo_fine || !kept_row))
          vo = sub(u.o, wo);
        if (ownz && ((owny >> i) & 1)) {
          if (lx.own_e)
            (fy ? eB1 : eB0)[rowE[i]] = kept_row ? u.e : ve;
          if (lx.own_o)
            (fy ? oB1 : oB0)[rowO[i]] = (kept_row && !lx.xo_fine) ? u.o : vo;
        }
      } else if (wout) {
        st_pair(wout + b * 64 + 2 * lane, R(0), R(0));
      }
      // x pass: output lane a from pairs a, a+1 and the even node of a+2
      const R o1 = __shfl_down_sync(0xffffffffu, vo, 1);
      R xv;
      if (!fz && !fy && ok) { // even taps are kept nodes: zero
        if constexpr (FAST)
          xv = fma(wx.w3, o1, wx.w1 * vo);
        else
          xv = stencil_eval<R, false>(sx, R(0), vo, R(0), o1, R(0));
      } else {
        const R e1 = __shfl_down_sync(0xffffffffu, ve, 1);
        const R e2 = __shfl_down_sync(0xffffffffu, ve, 2);
        if constexpr (FAST)
          xv = wx.eval(ve, vo, e1, o1, e2);
        else
          xv = stencil_eval<R, false>(sx, ve, vo, e1, o1, e2);
      }
      if (lane < 30)
        X[b * 32 + lane] = lx.xval ? xv : R(0);
    }
  };

  // ---- y pass weights (FAST: registers, rows j = warp + 8r)
  W5<R> wy[C::RW];
  __syncthreads(); // tables staged
  if constexpr (FAST) {
#pragma unroll
    for (int r = 0; r < C::RW; ++r) {
      const int j = warp + 8 * r;
      if (j < CY && cy0 + j < cy1)
        wy[r].load(sY[j]);
    }
  }
  auto y_eval = [&](int r) -> R {
    const int j = warp + 8 * r;
    const R *c = X + (2 * j) * 32 + lane;
    if constexpr (FAST)
      return wy[r].eval(c[0], c[32], c[64], c[96], c[128]);
    else
      return stencil_eval<R, false>(sY[j], c[0], c[32], c[64], c[96], c[128]);
  };
  auto y_all = [&](R *out) {
#pragma unroll
    for (int r = 0; r < C::RW; ++r) {
      const int j = warp + 8 * r;
      out[r] = (j < CY && cy0 + j < cy1) ? y_eval(r) : R(0);
    }
  };
  const uint32_t cxo = cx0 + lane;
  auto store_f = [&](uint32_t k, const R *v) {
#pragma unroll
    for (int r = 0; r < C::RW; ++r) {
      const int j = warp + 8 * r;
      if (j < CY && cy0 + j < cy1 && lx.xval)
        f[cxo + uint64_t(mx) * (cy0 + j) + mxy * k] = v[r];
    }
  };

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
      R gv[C::RW];
      y_all(gv);
      store_f(p, gv);
      __syncthreads();
    }
    cp_async_wait<0>();
    return;
  }

  // z refines: carried window c0,c1,c2 = G(pc-2), G(pc-1), G(pc)
  R c0[C::RW], c1[C::RW], c2[C::RW], zero[C::RW];
#pragma unroll
  for (int r = 0; r < C::RW; ++r)
    c0[r] = c1[r] = c2[r] = zero[r] = R(0);
  auto emit = [&](uint32_t k, const R *t0, const R *t1, const R *t2, const R *t3,
                  const R *t4) {
    if (k < cz0 || k >= cz1)
      return;
    R v[C::RW];
    if constexpr (FAST) {
      const Stencil<R> &s = sZ[k - cz0];
      const R w0 = s.w[0], w1 = s.w[1], w2 = s.w[2], w3 = s.w[3], w4 = s.w[4];
#pragma unroll
      for (int r = 0; r < C::RW; ++r) {
        R a = w0 * t0[r];
        a = fma(w1, t1[r], a);
        a = fma(w2, t2[r], a);
        a = fma(w3, t3[r], a);
        v[r] = fma(w4, t4[r], a);
      }
    } else {
#pragma unroll
      for (int r = 0; r < C::RW; ++r)
        v[r] = stencil_eval<R, false>(sZ[k - cz0], t0[r], t1[r], t2[r], t3[r], t4[r]);
    }
    store_f(k, v);
  };

  uint32_t pc = Z0; // last processed coarse plane
  uint32_t slot = 0;
  process_plane(pc, false, nullptr, nullptr, Wc);
  __syncthreads();
  y_all(c2);
  for (;;) {
    const uint32_t nxt = pc + 2 <= nz - 1 ? pc + 2 : pc + 1;
    if (nxt >= Z1)
      break;
    __syncthreads(); // X consumed before it is overwritten
    load_plane(issued++);
    load_plane(issued++);
    cp_async_wait<2>();
    __syncthreads();
    const uint32_t ns = slot ^ 1;
    process_plane(nxt, false, nullptr, nullptr, Wc + ns * C::PL);
    __syncthreads();
    R gn[C::RW], gf[C::RW];
    y_all(gn);
    if (nxt == pc + 2) { // the fine plane between the two coarse planes
      __syncthreads();
      process_plane(pc + 1, true, Wc + slot * C::PL, Wc + ns * C::PL, nullptr);
      __syncthreads();
      y_all(gf);
      emit(pc >> 1, c0, c1, c2, gf, gn); // q = pc: taps pc-2 .. pc+2
#pragma unroll
      for (int r = 0; r < C::RW; ++r) {
        c0[r] = c2[r];
        c1[r] = gf[r];
        c2[r] = gn[r];
      }
      pc = nxt;
      slot = ns;
    } else {
      // nxt = pc + 1 = nz - 1 (even nz): output pc/2 has no fine right
      // neighbour but mv(q) still reads position q+1 = nxt; the last output
      // (q = nz-1) reads positions q-1 = pc and q = nxt
      emit(pc >> 1, c0, c1, c2, gn, zero);
      emit((nxt + 1) >> 1, zero, c2, gn, zero, zero);
      pc = nxt;
      break;
    }
  }
  // last coarse plane of an odd extent: q = nz-1 = pc (right boundary form)
  if (pc == nz - 1 && (pc & 1) == 0)
    emit(pc >> 1, c0, c1, c2, zero, zero);
  cp_async_wait<0>();
}

} // namespace mgrg
