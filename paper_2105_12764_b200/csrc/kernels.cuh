// kernels.cuh -- the hand-written sm_100a kernels of the refactoring path.
//
//   dec_level_kernel  GPK (coefficients) + class-order store + packed coarse
//                     store + vec(C) masking + merged mass-trans R*M along
//                     x, y, z  ->  load vector f            (one HBM pass)
//   rec_load_kernel   class gather (vec(C)) + R*M along x, y, z -> f
//   rec_gpk_kernel    coarse' (= a_{l-1} - z) + class -> a_l (GPK inverse)
//   thomas_x_kernel   batched Thomas along dim 0 (contiguous fibers,
//                     warp-transposed through shared memory)
//   thomas_strided_kernel  batched Thomas along dim 1/2 (thread per fiber,
//                     coalesced rows); both with the apply/unapply epilogue
//
// All of them are bandwidth-bound stencil / recurrence / permutation work:
// no tensor cores (no dense contraction anywhere).
#pragma once

#include "common.cuh"
#include "level.cuh"

namespace mgrg {

// ---------------------------------------------------------------------------
// Per-dimension tile geometry.  A CTA owns C coarse outputs [c0, c1) along a
// dimension; it reads the fine box [lo, hi) (reach 2 of the merged stencil,
// which also covers the +-1 GPK corners of every fine node in the box) and
// owns (stores class / packed coarse values of) fine positions [olo, ohi).
// ---------------------------------------------------------------------------
struct Span {
  uint32_t c0, c1, lo, hi, olo, ohi;
};
__device__ __forceinline__ Span make_span(uint32_t c0, uint32_t C, uint32_t n,
                                          uint32_t m, bool refine) {
  Span s;
  s.c0 = c0;
  s.c1 = min(c0 + C, m);
  if (refine) {
    s.lo = c0 ? 2 * c0 - 2 : 0;
    s.hi = min(n, 2 * s.c1 + 1);
    s.olo = 2 * c0;
    s.ohi = s.c1 == m ? n : 2 * s.c1;
  } else {
    s.lo = c0;
    s.hi = s.c1;
    s.olo = c0;
    s.ohi = s.c1;
  }
  return s;
}

template <typename R>
__device__ __forceinline__ uint64_t class_slot(const LevelGeom<R> &g, unsigned mask,
                                               uint32_t px, uint32_t py,
                                               uint32_t pz) {
  // class_slot (grid.hpp:149-164) on the padded 3-D lattice
  const uint32_t wx = (mask & 1) ? fine_rank(px) : coarse_rank(px);
  const uint32_t wy = (mask & 2) ? fine_rank(py) : coarse_rank(py);
  const uint32_t wz = (mask & 4) ? fine_rank(pz) : coarse_rank(pz);
  return g.tbase[mask] + wx + uint64_t(g.tex[mask]) * (wy + uint64_t(g.tey[mask]) * wz);
}

// Multilinear interpolation of a fine node from its coarse corners
// (interpolate_node, kernels.hpp:193-223): lowest fine dimension first.
// c(dx, dy, dz) returns the corner value at offset (dx, dy, dz) in {-1,0,1}.
template <typename R, typename C>
__device__ __forceinline__ R interp_node(C &&c, unsigned mask, R tx, R ty, R tz) {
  switch (mask) {
  case 1:
    return lerp(c(-1, 0, 0), c(1, 0, 0), tx);
  case 2:
    return lerp(c(0, -1, 0), c(0, 1, 0), ty);
  case 4:
    return lerp(c(0, 0, -1), c(0, 0, 1), tz);
  case 3:
    return lerp(lerp(c(-1, -1, 0), c(1, -1, 0), tx),
                lerp(c(-1, 1, 0), c(1, 1, 0), tx), ty);
  case 5:
    return lerp(lerp(c(-1, 0, -1), c(1, 0, -1), tx),
                lerp(c(-1, 0, 1), c(1, 0, 1), tx), tz);
  case 6:
    return lerp(lerp(c(0, -1, -1), c(0, 1, -1), ty),
                lerp(c(0, -1, 1), c(0, 1, 1), ty), tz);
  default: {
    const R a = lerp(lerp(c(-1, -1, -1), c(1, -1, -1), tx),
                     lerp(c(-1, 1, -1), c(1, 1, -1), tx), ty);
    const R b = lerp(lerp(c(-1, -1, 1), c(1, -1, 1), tx),
                     lerp(c(-1, 1, 1), c(1, 1, 1), tx), ty);
    return lerp(a, b, tz);
  }
  }
}

template <int CX, int CY> struct TileCfg {
  static constexpr int T = CX * CY;
  static constexpr int BXM = 2 * CX + 3; // odd: conflict-free row pitch
  static constexpr int BYM = 2 * CY + 3;
  static constexpr int PLANE = BXM * BYM;
};

template <typename R, int CX, int CY> constexpr size_t dec_level_smem() {
  using C = TileCfg<CX, CY>;
  return sizeof(R) * (5 * C::PLANE + C::BYM * CX + 5 * CY * CX);
}
template <typename R, int CX, int CY> constexpr size_t rec_load_smem() {
  using C = TileCfg<CX, CY>;
  return sizeof(R) * (3 * C::PLANE + C::BYM * CX + 5 * CY * CX);
}
template <typename R, int CX, int CY> constexpr size_t rec_gpk_smem() {
  return sizeof(R) * 3 * (CX + 1) * (CY + 1);
}

// x then y merged mass-trans of one staged plane V (box coordinates) into
// G[slot] for this thread's (ti, tj) output column.  Returns the value.
template <typename R, int CX, int CY>
__device__ __forceinline__ void xy_masstrans(const LevelGeom<R> &g, const R *V,
                                             R *X, const Span &sx,
                                             const Span &sy, int tid, R *gout) {
  using C = TileCfg<CX, CY>;
  const bool rx = g.refine & 1, ry = g.refine & 2;
  const uint32_t BY = sy.hi - sy.lo;
  // x pass: every box row -> CX coarse-x outputs
  for (int e = tid; e < int(BY) * CX; e += C::T) {
    const int by = e / CX, i = e - by * CX;
    const uint32_t cx = sx.c0 + i;
    if (cx < sx.c1) {
      const R *row = V + by * C::BXM;
      R v;
      if (rx) {
        const uint32_t q = coarse_pos(cx, g.n[0]);
        v = masstrans_at<R>([&](uint32_t j) { return row[j - sx.lo]; }, q, g.n[0],
                            g.h[0], g.r[0]);
      } else {
        v = row[cx - sx.lo];
      }
      X[by * CX + i] = v;
    }
  }
  __syncthreads();
  // y pass: this thread's column
  const int ti = tid % CX, tj = tid / CX;
  const uint32_t cx = sx.c0 + ti, cy = sy.c0 + tj;
  if (cx < sx.c1 && cy < sy.c1) {
    R v;
    if (ry) {
      const uint32_t q = coarse_pos(cy, g.n[1]);
      v = masstrans_at<R>([&](uint32_t j) { return X[(j - sy.lo) * CX + ti]; }, q,
                          g.n[1], g.h[1], g.r[1]);
    } else {
      v = X[(cy - sy.lo) * CX + ti];
    }
    *gout = v;
  }
}

// z stage: G ring of the last five planes (per thread), emits f rows.
template <typename R, int CX, int CY>
__device__ __forceinline__ void z_emit(const LevelGeom<R> &g, const R *G,
                                       uint32_t pz, uint32_t &kk, uint32_t kend,
                                       int tid, bool valid, R *__restrict__ f,
                                       uint64_t fcol) {
  using C = TileCfg<CX, CY>;
  const uint32_t nz = g.n[2];
  const uint64_t fplane = uint64_t(g.m[0]) * g.m[1];
  if (!(g.refine & 4)) {
    // identity along z: plane pz is coarse output pz
    if (valid)
      f[fcol + fplane * pz] = G[(pz % 5) * C::T + tid];
    kk = pz + 1;
    return;
  }
  while (kk < kend) {
    const uint32_t q = coarse_pos(kk, nz);
    const uint32_t need = min(q + 2, nz - 1);
    if (need > pz)
      break;
    if (valid) {
      const R v = masstrans_at<R>([&](uint32_t j) { return G[(j % 5) * C::T + tid]; },
                                  q, nz, g.h[2], g.r[2]);
      f[fcol + fplane * kk] = v;
    }
    ++kk;
  }
}

// ---------------------------------------------------------------------------
// Decompose, one level (refactor.hpp:165-175 minus the solves):
//   GPK forward on the level-l array `in` (kernels.hpp:231-279),
//   class l store in class order (refactor.hpp:273-281 fused copy),
//   packed kept-node values -> P (the a_{l-1} buffer, apply adds z later),
//   vec(C) + merged R*M along x, y, z -> f (refactor.hpp:251-346).
// Grid: (ceil(mx/CX), ceil(my/CY), ceil(mz/zchunk)); the CTA marches its
// z-chunk one fine plane at a time with a 4-plane LDGSTS ring.
// ---------------------------------------------------------------------------
template <typename R, int CX, int CY>
__global__ void __launch_bounds__(CX *CY)
    dec_level_kernel(LevelGeom<R> g, const R *__restrict__ in, R *__restrict__ cls,
                     R *__restrict__ P, R *__restrict__ f, uint32_t zchunk) {
  using C = TileCfg<CX, CY>;
  extern __shared__ __align__(16) unsigned char smem_bytes[];
  R *raw = reinterpret_cast<R *>(smem_bytes); // [4][BYM][BXM]
  R *V = raw + 4 * C::PLANE;                   // [BYM][BXM]
  R *X = V + C::PLANE;                         // [BYM][CX]
  R *G = X + C::BYM * CX;                      // [5][T]

  const int tid = threadIdx.x;
  const uint32_t nx = g.n[0], ny = g.n[1], nz = g.n[2];
  const uint32_t mx = g.m[0], my = g.m[1];
  const Span sx = make_span(blockIdx.x * CX, CX, nx, g.m[0], g.refine & 1);
  const Span sy = make_span(blockIdx.y * CY, CY, ny, g.m[1], g.refine & 2);
  const Span sz = make_span(blockIdx.z * zchunk, zchunk, nz, g.m[2], g.refine & 4);
  const uint32_t BX = sx.hi - sx.lo, BY = sy.hi - sy.lo, NB = BX * BY;
  const uint64_t nxy = uint64_t(nx) * ny;

  auto load_plane = [&](uint32_t pz) {
    R *dst = raw + (pz & 3) * C::PLANE;
    const R *src = in + nxy * pz + uint64_t(sy.lo) * nx + sx.lo;
    for (uint32_t e = tid; e < NB; e += C::T) {
      const uint32_t by = e / BX, bx = e - by * BX;
      cp_async(dst + by * C::BXM + bx, src + uint64_t(by) * nx + bx);
    }
  };

  load_plane(sz.lo);
  cp_async_commit();
  if (sz.lo + 1 < sz.hi)
    load_plane(sz.lo + 1);
  cp_async_commit();

  const int ti = tid % CX, tj = tid / CX;
  const bool valid = (sx.c0 + ti < sx.c1) && (sy.c0 + tj < sy.c1);
  const uint64_t fcol = (sx.c0 + ti) + uint64_t(mx) * (sy.c0 + tj);
  uint32_t kk = sz.c0;

  for (uint32_t pz = sz.lo; pz < sz.hi; ++pz) {
    if (pz + 2 < sz.hi)
      load_plane(pz + 2);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();

    // ---- GPK + class / packed-coarse stores + vec(C) -> V ----
    const bool fz = !is_coarse(pz, nz);
    const bool ownz = pz >= sz.olo && pz < sz.ohi;
    const R tz = fz ? __ldg(g.r[2] + pz - 1) : R(0);
    const R *p0 = raw + (pz & 3) * C::PLANE;
    const R *pm = raw + ((pz - 1) & 3) * C::PLANE;
    const R *pp = raw + ((pz + 1) & 3) * C::PLANE;
    for (uint32_t e = tid; e < NB; e += C::T) {
      const uint32_t by = e / BX, bx = e - by * BX;
      const uint32_t px = sx.lo + bx, py = sy.lo + by;
      const bool fx = !is_coarse(px, nx), fy = !is_coarse(py, ny);
      const unsigned mask = unsigned(fx) | (unsigned(fy) << 1) | (unsigned(fz) << 2);
      const int o = by * C::BXM + bx;
      const R u = p0[o];
      const bool own = ownz && px >= sx.olo && px < sx.ohi && py >= sy.olo && py < sy.ohi;
      R v;
      if (mask == 0) {
        v = R(0);
        if (own)
          P[coarse_rank(px) + uint64_t(mx) * (coarse_rank(py) + uint64_t(my) * coarse_rank(pz))] = u;
      } else {
        const R tx = fx ? __ldg(g.r[0] + px - 1) : R(0);
        const R ty = fy ? __ldg(g.r[1] + py - 1) : R(0);
        const R ip = interp_node<R>(
            [&](int dx, int dy, int dz) {
              const R *pl = dz < 0 ? pm : (dz > 0 ? pp : p0);
              return pl[o + dy * C::BXM + dx];
            },
            mask, tx, ty, tz);
        v = sub(u, ip);
        if (own)
          cls[class_slot(g, mask, px, py, pz)] = v;
      }
      V[o] = v;
    }
    __syncthreads();

    R gval = R(0);
    xy_masstrans<R, CX, CY>(g, V, X, sx, sy, tid, &gval);
    G[(pz % 5) * C::T + tid] = gval;
    z_emit<R, CX, CY>(g, G, pz, kk, sz.c1, tid, valid, f, fcol);
  }
}

// ---------------------------------------------------------------------------
// Recompose load vector, one level (refactor.hpp:191-195 flavour of
// masstrans_dim0 / masstrans_later): vec(C) built from class l (coarse nodes
// read as zero) and R*M along x, y, z -> f.  3-plane LDGSTS gather ring.
// ---------------------------------------------------------------------------
template <typename R, int CX, int CY>
__global__ void __launch_bounds__(CX *CY)
    rec_load_kernel(LevelGeom<R> g, const R *__restrict__ cls, R *__restrict__ f,
                    uint32_t zchunk) {
  using C = TileCfg<CX, CY>;
  extern __shared__ __align__(16) unsigned char smem_bytes[];
  R *Vr = reinterpret_cast<R *>(smem_bytes); // [3][BYM][BXM]
  R *X = Vr + 3 * C::PLANE;                   // [BYM][CX]
  R *G = X + C::BYM * CX;                     // [5][T]

  const int tid = threadIdx.x;
  const uint32_t nx = g.n[0], ny = g.n[1], nz = g.n[2];
  const uint32_t mx = g.m[0];
  const Span sx = make_span(blockIdx.x * CX, CX, nx, g.m[0], g.refine & 1);
  const Span sy = make_span(blockIdx.y * CY, CY, ny, g.m[1], g.refine & 2);
  const Span sz = make_span(blockIdx.z * zchunk, zchunk, nz, g.m[2], g.refine & 4);
  const uint32_t BX = sx.hi - sx.lo, BY = sy.hi - sy.lo, NB = BX * BY;

  auto load_plane = [&](uint32_t pz) {
    R *dst = Vr + (pz % 3) * C::PLANE;
    const bool fz = !is_coarse(pz, nz);
    for (uint32_t e = tid; e < NB; e += C::T) {
      const uint32_t by = e / BX, bx = e - by * BX;
      const uint32_t px = sx.lo + bx, py = sy.lo + by;
      const unsigned mask = unsigned(!is_coarse(px, nx)) |
                            (unsigned(!is_coarse(py, ny)) << 1) | (unsigned(fz) << 2);
      R *d = dst + by * C::BXM + bx;
      if (mask == 0)
        *d = R(0);
      else
        cp_async(d, cls + class_slot(g, mask, px, py, pz));
    }
  };

  load_plane(sz.lo);
  cp_async_commit();
  if (sz.lo + 1 < sz.hi)
    load_plane(sz.lo + 1);
  cp_async_commit();

  const int ti = tid % CX, tj = tid / CX;
  const bool valid = (sx.c0 + ti < sx.c1) && (sy.c0 + tj < sy.c1);
  const uint64_t fcol = (sx.c0 + ti) + uint64_t(mx) * (sy.c0 + tj);
  uint32_t kk = sz.c0;

  for (uint32_t pz = sz.lo; pz < sz.hi; ++pz) {
    if (pz + 2 < sz.hi)
      load_plane(pz + 2);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    R gval = R(0);
    xy_masstrans<R, CX, CY>(g, Vr + (pz % 3) * C::PLANE, X, sx, sy, tid, &gval);
    G[(pz % 5) * C::T + tid] = gval;
    z_emit<R, CX, CY>(g, G, pz, kk, sz.c1, tid, valid, f, fcol);
  }
}

// ---------------------------------------------------------------------------
// Recompose GPK inverse, one level (refactor.hpp:198-200): coarse nodes of
// a_l take the packed coarse' values (unapply_expand), fine nodes take
// interp(coarse') + class (scatter_class + gpk inverse).  cls == nullptr:
// classes above classes_used, read as zero (refactor.hpp:192, 439).
// Grid: (ceil(mx/CX), ceil(my/CY), ceil(mz/zchunk)) over coarse ranks.
// ---------------------------------------------------------------------------
template <typename R, int CX, int CY>
__global__ void __launch_bounds__(CX *CY)
    rec_gpk_kernel(LevelGeom<R> g, const R *__restrict__ coarse,
                   const R *__restrict__ cls, R *__restrict__ out, uint32_t zchunk) {
  constexpr int T = CX * CY, PX = CX + 1, PY = CY + 1, PL = PX * PY;
  extern __shared__ __align__(16) unsigned char smem_bytes[];
  R *Cs = reinterpret_cast<R *>(smem_bytes); // [3][PY][PX]

  const int tid = threadIdx.x;
  const uint32_t nx = g.n[0], ny = g.n[1], nz = g.n[2];
  const uint32_t mx = g.m[0], my = g.m[1], mz = g.m[2];
  const bool rz = g.refine & 4;
  const Span sx = make_span(blockIdx.x * CX, CX, nx, mx, g.refine & 1);
  const Span sy = make_span(blockIdx.y * CY, CY, ny, my, g.refine & 2);
  const uint32_t kz0 = blockIdx.z * zchunk, kz1 = min(kz0 + zchunk, mz);
  // coarse ranks staged: [c0, c0 + C + 1) clipped
  const uint32_t CXn = min(sx.c0 + CX + 1, mx) - sx.c0;
  const uint32_t CYn = min(sy.c0 + CY + 1, my) - sy.c0;
  const uint32_t NC = CXn * CYn;
  const uint64_t mxy = uint64_t(mx) * my;
  const uint32_t OXN = sx.ohi - sx.olo, OYN = sy.ohi - sy.olo, NO = OXN * OYN;
  const uint64_t nxy = uint64_t(nx) * ny;

  auto load_plane = [&](uint32_t k) {
    R *dst = Cs + (k % 3) * PL;
    const R *src = coarse + mxy * k + uint64_t(sy.c0) * mx + sx.c0;
    for (uint32_t e = tid; e < NC; e += T) {
      const uint32_t j = e / CXn, i = e - j * CXn;
      cp_async(dst + j * PX + i, src + uint64_t(j) * mx + i);
    }
  };
  const uint32_t klast = min(kz1 + 1, mz); // planes needed: [kz0, klast)
  load_plane(kz0);
  cp_async_commit();
  if (kz0 + 1 < klast)
    load_plane(kz0 + 1);
  cp_async_commit();

  auto emit_plane = [&](uint32_t pz, const R *clo, const R *chi, bool fz, R tz) {
    R *orow = out + nxy * pz;
    for (uint32_t e = tid; e < NO; e += T) {
      const uint32_t oy = e / OXN, ox = e - oy * OXN;
      const uint32_t px = sx.olo + ox, py = sy.olo + oy;
      const bool fx = !is_coarse(px, nx), fy = !is_coarse(py, ny);
      const unsigned mask = unsigned(fx) | (unsigned(fy) << 1) | (unsigned(fz) << 2);
      // local coarse ranks of the lower corner (fine) or the node (coarse)
      const uint32_t lx = (fx ? fine_rank(px) : coarse_rank(px)) - sx.c0;
      const uint32_t ly = (fy ? fine_rank(py) : coarse_rank(py)) - sy.c0;
      R v;
      if (mask == 0) {
        v = clo[ly * PX + lx];
      } else {
        const R c = cls ? __ldg(cls + class_slot(g, mask, px, py, pz)) : R(0);
        const R tx = fx ? __ldg(g.r[0] + px - 1) : R(0);
        const R ty = fy ? __ldg(g.r[1] + py - 1) : R(0);
        const R ip = interp_node<R>(
            [&](int dx, int dy, int dz) {
              const R *pl = dz > 0 ? chi : clo;
              const uint32_t ix = lx + (dx > 0), iy = ly + (dy > 0);
              return pl[iy * PX + ix];
            },
            mask, tx, ty, tz);
        v = add(ip, c);
      }
      orow[uint64_t(py) * nx + px] = v;
    }
  };

  for (uint32_t k = kz0; k < kz1; ++k) {
    if (k + 2 < klast)
      load_plane(k + 2);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const R *clo = Cs + (k % 3) * PL;
    const uint32_t pz = rz ? coarse_pos(k, nz) : k;
    emit_plane(pz, clo, clo, false, R(0));
    if (rz && pz + 1 < nz - 1) // the fine plane between coarse k and k+1
      emit_plane(pz + 1, clo, Cs + ((k + 1) % 3) * PL, true, __ldg(g.r[2] + pz));
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Thomas solves (thomas_fiber, kernels.hpp:143-151), batched over fibers.
// ---------------------------------------------------------------------------
template <typename R>
__device__ __forceinline__ void epi_store(Epi epi, R *f, const R *base, R *out, uint64_t idx,
                                          R z) {
  if (epi == Epi::none)
    f[idx] = z;
  else if (epi == Epi::add)
    out[idx] = add(base[idx], z); // apply_pack: a + w (refactor.hpp:388)
  else
    out[idx] = sub(base[idx], z); // unapply_expand: a - w (refactor.hpp:416)
}

// Fibers along a strided dimension (stride S elements, length t.m); fiber k
// starts at (k % inner) + (k / inner) * ostride.  One thread per fiber, so a
// warp touches 32 consecutive x positions per step (coalesced).  The forward
// sweep writes its partial results back in place (L2-resident for the
// backward sweep, which reads them in reverse).
template <typename R, int B = 8>
__global__ void __launch_bounds__(128)
    thomas_strided_kernel(R *f, ThomasGeom<R> t, uint64_t S, uint32_t inner,
                          uint64_t ostride, uint64_t nfibers, Epi epi, const R *base, R *out) {
  pdl_wait();
  // f, base and out may alias (the epilogues write in place): no __restrict__
  const uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= nfibers)
    return;
  const uint32_t M = t.m;
  const uint64_t st = (k % inner) + (k / inner) * ostride;
  R *fp = f + st;
  R v = fp[0];
  for (uint32_t i0 = 1; i0 < M; i0 += B) {
    R buf[B];
#pragma unroll
    for (int b = 0; b < B; ++b)
      if (i0 + b < M)
        buf[b] = fp[uint64_t(i0 + b) * S];
#pragma unroll
    for (int b = 0; b < B; ++b)
      if (i0 + b < M) {
        v = add(buf[b], mul(__ldg(t.fwd + i0 + b), v));
        if (i0 + b < M - 1)
          fp[uint64_t(i0 + b) * S] = v;
      }
  }
  v = mul(v, __ldg(t.ip + M - 1));
  epi_store(epi, f, base, out, st + uint64_t(M - 1) * S, v);
  const bool ep = epi != Epi::none;
  for (int32_t i0 = int32_t(M) - 2; i0 >= 0; i0 -= B) {
    R buf[B], bb[B];
    // the batch's solution inputs and (last solve) epilogue bases together
#pragma unroll
    for (int b = 0; b < B; ++b)
      if (i0 - b >= 0) {
        buf[b] = fp[uint64_t(i0 - b) * S];
        bb[b] = ep ? base[st + uint64_t(i0 - b) * S] : R(0);
      }
#pragma unroll
    for (int b = 0; b < B; ++b)
      if (i0 - b >= 0) {
        const uint32_t i = i0 - b;
        v = mul(sub(buf[b], mul(__ldg(t.h + i), v)), __ldg(t.ip + i));
        const uint64_t idx = st + uint64_t(i) * S;
        if (!ep)
          f[idx] = v;
        else
          out[idx] = epi == Epi::add ? add(bb[b], v) : sub(bb[b], v);
      }
  }
}

// Fibers along dim 0 (contiguous, length t.m, fiber k at k*t.m).  A warp owns
// 32 fibers and walks them in 32-element chunks: the chunk is loaded
// row-by-row (coalesced), transposed through a padded 32x33 shared tile,
// each lane runs the recurrence along its fiber, and the chunk is written
// back coalesced.
template <typename R>
__global__ void __launch_bounds__(128)
    thomas_x_kernel(R *f, ThomasGeom<R> t, uint64_t nfibers, Epi epi, const R *base,
                    R *out) { // f, base, out may alias
  __shared__ R tile_all[4][32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  auto tile = tile_all[w];
  const uint64_t fb0 = (uint64_t(blockIdx.x) * 4 + w) * 32;
  if (fb0 >= nfibers)
    return;
  const uint32_t M = t.m;
  const uint32_t nch = (M + 31) / 32;
  const uint32_t nf = nfibers - fb0 < 32 ? uint32_t(nfibers - fb0) : 32u;
  R v = R(0);
  // forward sweep
  for (uint32_t c = 0; c < nch; ++c) {
    const uint32_t j = c * 32 + lane;
    for (uint32_t fr = 0; fr < nf; ++fr)
      if (j < M)
        tile[fr][lane] = f[(fb0 + fr) * M + j];
    __syncwarp();
    for (uint32_t jj = 0; jj < 32; ++jj) {
      const uint32_t jg = c * 32 + jj;
      if (jg >= M)
        break;
      const R x = tile[lane][jj];
      v = jg == 0 ? x : add(x, mul(__ldg(t.fwd + jg), v));
      if (jg == M - 1)
        v = mul(v, __ldg(t.ip + M - 1));
      tile[lane][jj] = v;
    }
    __syncwarp();
    for (uint32_t fr = 0; fr < nf; ++fr)
      if (j < M) {
        if (j == M - 1)
          epi_store(epi, f, base, out, (fb0 + fr) * M + j, tile[fr][lane]);
        else
          f[(fb0 + fr) * M + j] = tile[fr][lane];
      }
    __syncwarp();
  }
  // backward sweep (v holds z_{M-1})
  for (int32_t c = int32_t(nch) - 1; c >= 0; --c) {
    const uint32_t j = c * 32 + lane;
    for (uint32_t fr = 0; fr < nf; ++fr)
      if (j < M - 1)
        tile[fr][lane] = f[(fb0 + fr) * M + j];
    __syncwarp();
    for (int32_t jj = 31; jj >= 0; --jj) {
      const uint32_t jg = c * 32 + jj;
      if (jg >= M - 1)
        continue;
      v = mul(sub(tile[lane][jj], mul(__ldg(t.h + jg), v)), __ldg(t.ip + jg));
      tile[lane][jj] = v;
    }
    __syncwarp();
    for (uint32_t fr = 0; fr < nf; ++fr)
      if (j < M - 1)
        epi_store(epi, f, base, out, (fb0 + fr) * M + j, tile[fr][lane]);
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Unit-level kernels (kernels.hpp public API) for parity tests and callers
// of the standalone operators.  Simple one-thread-per-element forms.
// ---------------------------------------------------------------------------

// compute_coefficients / restore_coefficients, in place (kernels.hpp:284-310).
// Kept nodes are never written, so reading corners in place is race-free.
template <typename R>
__global__ void gpk_inplace_kernel(LevelGeom<R> g, R *a, int inverse) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t nx = g.n[0], ny = g.n[1], nz = g.n[2];
  if (i >= uint64_t(nx) * ny * nz)
    return;
  const uint32_t px = i % nx, py = (i / nx) % ny, pz = i / (uint64_t(nx) * ny);
  const bool fx = !is_coarse(px, nx), fy = !is_coarse(py, ny), fz = !is_coarse(pz, nz);
  const unsigned mask = unsigned(fx) | (unsigned(fy) << 1) | (unsigned(fz) << 2);
  if (!mask)
    return;
  const R tx = fx ? g.r[0][px - 1] : R(0), ty = fy ? g.r[1][py - 1] : R(0),
          tz = fz ? g.r[2][pz - 1] : R(0);
  const int64_t sy = nx, sz = int64_t(nx) * ny;
  const R ip = interp_node<R>(
      [&](int dx, int dy, int dz) { return a[int64_t(i) + dx + dy * sy + dz * sz]; },
      mask, tx, ty, tz);
  a[i] = inverse ? add(ip, a[i]) : sub(a[i], ip);
}

// masstrans_apply along `dim` (kernels.hpp:328-412).  ext: input extents,
// ext[dim] = n (level-l), output extents the same with ext[dim] = m.  dim 0
// reads its input in vec(C) form (kept nodes of the level-l lattice as 0).
template <typename R>
__global__ void masstrans_kernel(LevelGeom<R> g, int dim, uint32_t e0, uint32_t e1,
                                 uint32_t e2, const R *in, R *out) {
  const uint32_t ext[3] = {e0, e1, e2};
  uint32_t oext[3] = {e0, e1, e2};
  const uint32_t n = g.n[dim], m = g.m[dim];
  oext[dim] = m;
  const uint64_t total = uint64_t(oext[0]) * oext[1] * oext[2];
  const uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= total)
    return;
  uint32_t p[3];
  p[0] = idx % oext[0];
  p[1] = (idx / oext[0]) % oext[1];
  p[2] = idx / (uint64_t(oext[0]) * oext[1]);
  const uint64_t istr[3] = {1, ext[0], uint64_t(ext[0]) * ext[1]};
  const uint32_t i = p[dim];
  uint64_t base = 0;
  for (int d = 0; d < 3; ++d)
    if (d != dim)
      base += p[d] * istr[d];
  if (!((g.refine >> dim) & 1)) {
    out[idx] = in[base + uint64_t(i) * istr[dim]];
    return;
  }
  bool row_fine = false;
  if (dim == 0)
    for (int d = 1; d < 3; ++d)
      row_fine = row_fine || !is_coarse(p[d], g.n[d]);
  auto rd = [&](uint32_t j) -> R {
    const R v = in[base + uint64_t(j) * istr[dim]];
    if (dim == 0 && !row_fine && is_coarse(j, n))
      return R(0);
    return v;
  };
  out[idx] = masstrans_at<R>(rd, coarse_pos(i, n), n, g.h[dim], g.r[dim]);
}

// Fused class copy of masstrans_apply(dim 0, fused_copy): coefficient nodes
// of the level-l array -> class order (kernels.hpp:393-399).
template <typename R>
__global__ void class_copy_kernel(LevelGeom<R> g, const R *in, R *coef) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t nx = g.n[0], ny = g.n[1], nz = g.n[2];
  if (i >= uint64_t(nx) * ny * nz)
    return;
  const uint32_t px = i % nx, py = (i / nx) % ny, pz = i / (uint64_t(nx) * ny);
  const unsigned mask = unsigned(!is_coarse(px, nx)) |
                        (unsigned(!is_coarse(py, ny)) << 1) |
                        (unsigned(!is_coarse(pz, nz)) << 2);
  if (mask)
    coef[class_slot(g, mask, px, py, pz)] = in[i];
}

template <typename R>
__global__ void apply_kernel(uint64_t count, R *v, const R *z, int sign) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < count)
    v[i] = sign >= 0 ? add(v[i], z[i]) : sub(v[i], z[i]);
}

// reorder (grid.hpp:177-196 via make_layout_map, grid.cpp:167-221):
// hierarchical slot k -> natural offset of the level-l array.
template <typename R>
__global__ void reorder_kernel(LevelGeom<R> g, int to_natural, const R *in, R *out) {
  const uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t nx = g.n[0], ny = g.n[1];
  const uint64_t total = g.nodes(), ncoarse = g.coarse_nodes();
  if (k >= total)
    return;
  uint32_t p[3];
  if (k < ncoarse) {
    const uint32_t r0 = k % g.m[0], r1 = (k / g.m[0]) % g.m[1],
                   r2 = k / (uint64_t(g.m[0]) * g.m[1]);
    p[0] = coarse_pos(r0, nx);
    p[1] = coarse_pos(r1, ny);
    p[2] = coarse_pos(r2, g.n[2]);
  } else {
    const uint64_t c = k - ncoarse;
    // class bases ascend with the mask; empty types share the next base, so
    // the owning type is the first one whose end lies beyond c
    unsigned mask = 7;
    for (unsigned mm = 1; mm < 7; ++mm)
      if (c < g.tbase[mm + 1]) {
        mask = mm;
        break;
      }
    const uint64_t w = c - g.tbase[mask];
    const uint32_t ex = g.tex[mask], ey = g.tey[mask];
    const uint32_t w0 = w % ex, w1 = (w / ex) % ey, w2 = w / (uint64_t(ex) * ey);
    p[0] = (mask & 1) ? 2 * w0 + 1 : coarse_pos(w0, nx);
    p[1] = (mask & 2) ? 2 * w1 + 1 : coarse_pos(w1, ny);
    p[2] = (mask & 4) ? 2 * w2 + 1 : coarse_pos(w2, g.n[2]);
  }
  const uint64_t off = p[0] + uint64_t(nx) * (p[1] + uint64_t(ny) * p[2]);
  if (to_natural)
    out[off] = in[k];
  else
    out[k] = in[off];
}

} // namespace mgrg
