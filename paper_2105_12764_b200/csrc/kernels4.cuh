// kernels4.cuh -- decompose level kernel, instruction-lean generation.
//
// Same work decomposition as kernels2/3 (lane a owns the fine pair
// (X0 + 2a, X0 + 2a + 1); x pass on warp shuffles, y pass through shared
// memory, z pass in registers; GPK as prolongation x -> y -> z, which is
// bit-identical to interpolate_node's corner reduction).  The ncu captures
// of the earlier generations were issue-bound (73-78 % issue-active at
// 3.7-4.7 warp instructions per fine element, DRAM at 20 %); this one is
// written against that budget:
//   * staging by 16-byte LDGSTS: each box row is fetched as the 16-byte
//     aligned superset of its 64 elements (row pitches such as 1025 put every
//     row at a different alignment), readers apply the per-row shift
//     (plane part + row part, both tabled); 4x fewer copy instructions and
//     no per-element address arithmetic;
//   * per-row class offsets (extent_x(type) * rank_y, plane independent) and
//     the y ratios live in a per-CTA shared table; per plane only four class
//     base pointers change;
//   * one plane-processing call site (a small state machine walks the
//     coarse/fine plane order), y and z weights in shared memory, so the
//     kernel fits 3 CTAs per SM without rematerialisation.
#pragma once

#include "kernels3.cuh"

namespace mgrg {

template <typename R> constexpr int cy4() { return sizeof(R) == 4 ? 18 : 8; }

template <typename R, int CY> struct T4 {
  static constexpr int NW = 8, T = 256;
  static constexpr int V = 16 / int(sizeof(R));   // elements per 16-byte chunk
  static constexpr int BYR = 2 * CY + 3;          // box rows
  static constexpr int NI = (BYR + NW - 1) / NW;  // rows per warp
  static constexpr int RW = (CY + NW - 1) / NW;   // y outputs per warp
  static constexpr int RP = 64 + V;               // raw row pitch (elements)
  static constexpr int NCH = RP / V;              // chunks per raw row
  static constexpr int RPL = BYR * RP;            // raw plane elements
  static constexpr int WPL = BYR * 64;            // W plane elements
  static constexpr int ZC = 32;                   // coarse-z outputs per CTA
  static constexpr int NCK = (BYR * NCH + T - 1) / T; // staging chunks per thread
};

template <typename R, int CY> constexpr size_t dec4_smem() {
  using C = T4<R, CY>;
  return al16(sizeof(R) * 4 * C::RPL) + al16(sizeof(R) * 2 * C::WPL) +
         al16(sizeof(R) * C::BYR * 32) + al16(sizeof(R) * 8 * CY) +
         al16(sizeof(R) * 8 * C::ZC) + al16(sizeof(Stencil<R>) * CY) +
         al16(sizeof(Stencil<R>) * C::ZC) + al16(sizeof(R) * (2 * C::ZC + 4)) +
         al16(sizeof(uint4) * C::BYR) + al16(sizeof(R) * C::BYR);
}

template <typename R, int CY, bool FAST, int MINB = 3>
__global__ void __launch_bounds__(256, MINB)
    dec4_kernel(LevelGeom<R> g, const Stencil<R> *__restrict__ stx,
                const Stencil<R> *__restrict__ sty, const Stencil<R> *__restrict__ stz,
                const R *__restrict__ in, R *__restrict__ cls, R *__restrict__ P,
                R *__restrict__ f, uint32_t ntx, uint32_t nty, uint32_t ntz) {
  using C = T4<R, CY>;
  using A = Arith<R, FAST>;
  extern __shared__ __align__(16) unsigned char smem_bytes[];
  Carve cv{smem_bytes};
  R *Uraw = cv.take<R>(4 * C::RPL);   // [4][BYR][RP] raw planes (shifted rows)
  R *Wc = cv.take<R>(2 * C::WPL);     // [2][BYR][64] W of the last two coarse planes
  R *X = cv.take<R>(C::BYR * 32);     // [BYR][32] x-pass results
  R *wY = cv.take<R>(8 * CY);         // FAST y weights, 8 per output row
  R *wZ = cv.take<R>(8 * C::ZC);      // FAST z weights
  Stencil<R> *sY = cv.take<Stencil<R>>(CY);    // exact y stencils
  Stencil<R> *sZ = cv.take<Stencil<R>>(C::ZC); // exact z stencils
  R *tzv = cv.take<R>(2 * C::ZC + 4);          // r_z of each box plane
  uint4 *rowT = cv.take<uint4>(C::BYR);        // {mx*wy, (nx-mx)*wy, shift_y, flags}
  R *tyT = cv.take<R>(C::BYR);                 // r_y of fine rows

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
  const uint32_t OZ0 = rz ? 2 * cz0 : cz0, OZ1 = rz ? (cz1 == mz ? nz : 2 * cz1) : cz1;
  const uint64_t nxy = uint64_t(nx) * ny;
  const uint64_t mxy = uint64_t(mx) * my;
  const uint64_t ntot = nxy * nz;

  // ---- per-CTA tables
  {
    const uint32_t nyo = cy1 - cy0;
    stage_stencils(sY, sty + cy0, nyo, tid);
    if (rz)
      stage_stencils(sZ, stz + cz0, cz1 - cz0, tid);
    if constexpr (FAST) {
      for (uint32_t e = tid; e < 8 * nyo; e += 256)
        wY[e] = (e & 7) < 5 ? sty[cy0 + (e >> 3)].w[e & 7] : R(0);
      if (rz)
        for (uint32_t e = tid; e < 8 * (cz1 - cz0); e += 256)
          wZ[e] = (e & 7) < 5 ? stz[cz0 + (e >> 3)].w[e & 7] : R(0);
    }
    if (rz)
      for (uint32_t p = Z0 + tid; p < Z1; p += 256)
        tzv[p - Z0] = ((p & 1) && p < nz - 1) ? g.r[2][p - 1] : R(0);
    const uint32_t OY0 = 2 * cy0, OY1 = cy1 == my ? ny : 2 * cy1;
    for (int b = tid; b < C::BYR; b += 256) {
      const int y = Y0 + b;
      const bool ok = y >= 0 && y < int(ny);
      const bool fy = ok && (y & 1) && y < int(ny) - 1;
      const uint32_t wy = ok ? (fy ? uint32_t(y) >> 1 : (uint32_t(y) + 1) >> 1) : 0;
      const uint32_t own = ok && uint32_t(y) >= OY0 && uint32_t(y) < OY1;
      const uint32_t shy = uint32_t((int64_t(y) * int64_t(nx)) & (C::V - 1));
      rowT[b] = make_uint4(mx * wy, (nx - mx) * wy, shy,
                           uint32_t(ok) | (uint32_t(fy) << 1) | (own << 2));
      tyT[b] = fy ? g.r[1][y - 1] : R(0);
    }
  }

  // ---- per-lane x geometry and x stencil (registers)
  const LaneX<R> lx = lane_x(g, lane, cx0, cx1);
  const Stencil<R> sx = stx[min(cx0 + min(uint32_t(lane), 29u), mx - 1)];
  W5<R> wx;
  if constexpr (FAST)
    wx.load(sx);

  // ---- 16-byte staging.  Box row b, chunk c covers elements
  // [al(b) + c*V, al(b) + c*V + V) with al(b) = (rowstart(b) & ~(V-1)),
  // rowstart(b) = p*nxy + (Y0+b)*nx + X0.
  auto load_plane = [&](uint32_t p) {
    if (p < Z1) {
      R *dst = Uraw + (p & 3) * C::RPL;
      const int64_t pbase = int64_t(p) * int64_t(nxy) + X0;
#pragma unroll
      for (int k = 0; k < C::NCK; ++k) {
        const int e = tid + 256 * k;
        if (e < C::BYR * C::NCH) {
          const int b = e / C::NCH, c = e - b * C::NCH;
          const int y = Y0 + b;
          if (y >= 0 && y < int(ny)) {
            const int64_t rs = pbase + int64_t(y) * nx;
            const int64_t a = (rs & ~int64_t(C::V - 1)) + int64_t(c) * C::V;
            R *d = dst + b * C::RP + c * C::V;
            if (a >= 0 && a + C::V <= int64_t(ntot)) {
              cp_async16(d, in + a);
            } else {
#pragma unroll
              for (int v = 0; v < C::V; ++v)
                if (a + v >= 0 && a + v < int64_t(ntot))
                  cp_async(d + v, in + a + v);
            }
          }
        }
      }
    }
    cp_async_commit();
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
  auto y_all = [&](R *out) {
#pragma unroll
    for (int r = 0; r < C::RW; ++r) {
      const int j = warp + 8 * r;
      R v = R(0);
      if (j < CY && cy0 + j < cy1) {
        const R *c = X + (2 * j) * 32 + lane;
        if constexpr (FAST) {
          const R *w = wY + 8 * j;
          R a = w[0] * c[0];
          a = fma(w[1], c[32], a);
          a = fma(w[2], c[64], a);
          a = fma(w[3], c[96], a);
          v = fma(w[4], c[128], a);
        } else {
          v = stencil_eval<R, false>(sY[j], c[0], c[32], c[64], c[96], c[128]);
        }
      }
      out[r] = v;
    }
  };
  auto emit = [&](uint32_t k, const R *t0, const R *t1, const R *t2, const R *t3,
                  const R *t4) {
    if (k < cz0 || k >= cz1)
      return;
    R v[C::RW];
#pragma unroll
    for (int r = 0; r < C::RW; ++r) {
      if constexpr (FAST) {
        const R *w = wZ + 8 * (k - cz0);
        R a = w[0] * t0[r];
        a = fma(w[1], t1[r], a);
        a = fma(w[2], t2[r], a);
        a = fma(w[3], t3[r], a);
        v[r] = fma(w[4], t4[r], a);
      } else {
        v[r] = stencil_eval<R, false>(sZ[k - cz0], t0[r], t1[r], t2[r], t3[r], t4[r]);
      }
    }
    store_f(k, v);
  };

  __syncthreads(); // tables staged
  load_plane(Z0);
  load_plane(Z0 + 1);
  load_plane(Z0 + 2);
  uint32_t issued = Z0 + 3;

  // plane walk: Z0 (coarse), then (pc+2 coarse, pc+1 fine) pairs; with z
  // not refining every plane is coarse and emitted directly
  R c0[C::RW], c1[C::RW], c2[C::RW], gn[C::RW], zero[C::RW];
#pragma unroll
  for (int r = 0; r < C::RW; ++r)
    c0[r] = c1[r] = c2[r] = gn[r] = zero[r] = R(0);
  uint32_t pc = Z0, slot = 0;
  uint32_t p = Z0;
  bool fz = false;
  for (;;) {
    // ---- make plane p resident (coarse planes advance the prefetch)
    if (!fz) {
      if (p > Z0) {
        __syncthreads(); // X and the raw slots being refilled are consumed
        load_plane(issued++);
        if (rz)
          load_plane(issued++);
      }
      cp_async_wait<2>();
      __syncthreads();
    } else {
      __syncthreads(); // X consumed by the coarse plane's y pass
    }
    // ---- GPK + stores + x pass of plane p
    {
      const R *Up = Uraw + (p & 3) * C::RPL;
      const uint32_t ns = slot ^ 1;
      R *wout = fz ? nullptr : Wc + (p == Z0 ? 0 : ns) * C::WPL;
      const R *wlo = Wc + slot * C::WPL, *whi = Wc + ns * C::WPL;
      const R tz = fz ? tzv[p - Z0] : R(0);
      const bool ownz = p >= OZ0 && p < OZ1;
      const uint32_t wz = fz ? p >> 1 : (p + 1) >> 1;
      const uint32_t shp = uint32_t((int64_t(p) * int64_t(nxy) + X0) & (C::V - 1));
      const unsigned mzb = fz ? 4u : 0u;
      R *eB0 = fz ? cls + type_plane(g, mzb, wz) : P + mxy * wz;
      R *eB1 = cls + type_plane(g, mzb | 2u, wz);
      R *oB0 = lx.xo_fine ? cls + type_plane(g, mzb | 1u, wz) : eB0;
      R *oB1 = lx.xo_fine ? cls + type_plane(g, mzb | 3u, wz) : eB1;
#pragma unroll
      for (int i = 0; i < C::NI; ++i) {
        const int b = warp + 8 * i;
        if (b >= C::BYR)
          break;
        const uint4 rt = rowT[b];
        const bool ok = rt.w & 1, fy = rt.w & 2;
        const uint32_t sh = (shp + rt.z) & (C::V - 1);
        auto raw = [&](int bb, uint32_t s) -> Pair<R> {
          const R *q = Up + bb * C::RP + s + 2 * lane;
          if (s & 1)
            return {q[0], q[1]};
          return ld_pair(q);
        };
        R ve = R(0), vo = R(0);
        const bool kept_row = !fz && !fy;
        if (ok) {
          const Pair<R> u = raw(b, sh);
          R we, wo;
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
            const uint32_t shm = (shp + rowT[b - 1].z) & (C::V - 1);
            const uint32_t shq = (shp + rowT[b + 1].z) & (C::V - 1);
            const Pair<R> um = raw(b - 1, shm), up = raw(b + 1, shq);
            const R umn = __shfl_down_sync(0xffffffffu, um.e, 1);
            const R upn = __shfl_down_sync(0xffffffffu, up.e, 1);
            const R wmo = lx.xo_fine ? A::lerp(um.e, umn, lx.tx) : um.o;
            const R wpo = lx.xo_fine ? A::lerp(up.e, upn, lx.tx) : up.o;
            const R ty = tyT[b];
            we = A::lerp(um.e, up.e, ty);
            wo = A::lerp(wmo, wpo, ty);
          }
          if (wout)
            st_pair(wout + b * 64 + 2 * lane, we, wo);
          if (!kept_row && lx.xe_ok)
            ve = sub(u.e, we);
          if (lx.xo_ok && (lx.xo_fine || !kept_row))
            vo = sub(u.o, wo);
          if (ownz && (rt.w & 4)) {
            if (lx.own_e)
              (fy ? eB1 : eB0)[rt.x + lx.cr_e] = kept_row ? u.e : ve;
            if (lx.own_o)
              (fy ? oB1 : oB0)[(lx.xo_fine ? rt.y : rt.x) + lx.rk_o] =
                  (kept_row && !lx.xo_fine) ? u.o : vo;
          }
        } else if (wout) {
          st_pair(wout + b * 64 + 2 * lane, R(0), R(0));
        }
        // x pass: output lane a from pairs a, a+1 and the even node of a+2
        const R o1 = __shfl_down_sync(0xffffffffu, vo, 1);
        R xv;
        if (kept_row && ok) { // even taps are kept nodes: zero
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
    }
    __syncthreads(); // X complete
    // ---- y pass and z stage
    if (!rz) {
      R gv[C::RW];
      y_all(gv);
      store_f(p, gv);
      if (++p >= Z1)
        break;
      continue;
    }
    if (p == Z0) {
      y_all(c2);
    } else if (!fz) {
      y_all(gn);
      if (p == pc + 2) { // the fine plane between comes next
        fz = true;
        p = pc + 1;
        continue;
      }
      // p = pc + 1 = nz - 1 (even nz): output pc/2 has no fine right
      // neighbour but mv(q) still reads position q+1 = p; the last output
      // (q = nz-1) reads positions q-1 = pc and q = p
      emit(pc >> 1, c0, c1, c2, gn, zero);
      emit((p + 1) >> 1, zero, c2, gn, zero, zero);
      pc = p;
      break;
    } else {
      R gf[C::RW];
      y_all(gf);
      emit(pc >> 1, c0, c1, c2, gf, gn); // q = pc: taps pc-2 .. pc+2
#pragma unroll
      for (int r = 0; r < C::RW; ++r) {
        c0[r] = c2[r];
        c1[r] = gf[r];
        c2[r] = gn[r];
      }
      pc += 2;
      slot ^= 1;
      fz = false;
    }
    // next coarse plane
    const uint32_t nxt = pc + 2 <= nz - 1 ? pc + 2 : pc + 1;
    if (nxt >= Z1)
      break;
    p = nxt;
  }
  // last coarse plane of an odd extent: q = nz-1 = pc (right boundary form)
  if (rz && pc == nz - 1 && (pc & 1) == 0)
    emit(pc >> 1, c0, c1, c2, zero, zero);
  cp_async_wait<0>();
}

} // namespace mgrg
