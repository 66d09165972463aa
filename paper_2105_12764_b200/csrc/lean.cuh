// lean.cuh -- warp-tiled level kernels of the FAST policy for dyadic levels
// (every extent odd, so the coarse nodes are exactly the even positions).
//
// Why a separate family: the ncu captures of the pair-lane kernels
// (profiles/r01_*, r02_*) are issue-bound at 2-4 warp instructions per fine
// element with DRAM at 17-30 % of peak; their generality (even extents,
// per-row shifts, CTA-wide staging and barriers) costs the instructions.
// Here every warp is an independent tile and all per-row decisions are
// compile-time:
//   * lane a owns the coarse x column qc = 30*tx - 1 + a, i.e. the fine pair
//     (2qc, 2qc+1); lanes 1..30 produce outputs, lanes 0 and 31 are the
//     reach-2 halo of the merged R*M window;
//   * a row at fine (y, plane p) starts at p*n0*n1 + y*n0, whose parity is
//     (p + y) & 1 for odd n0, n1: the parity of every row of the unrolled
//     band is known at compile time, so every row is ONE 8/16-byte load per
//     lane (LDG.64/128), misaligned rows fetch (o_{a-1}, e_a) and take o_a
//     from the next lane;
//   * the warp walks a band of TY coarse rows (2TY+3 fine rows) through a
//     chunk of coarse planes, two fine planes per step (the even plane 2k,
//     then the odd plane 2k-1 between the last two even ones): GPK as
//     prolongation x -> y -> z with the even planes' interpolant W carried
//     in registers, merged R*M along x on shuffles, along y over the band's
//     rows in registers, along z as three rolling accumulators.
// No shared memory, no barriers; the level array, class buffer and load
// vector are touched once each (plus the band's 3 halo rows, L2-resident).
#pragma once

#include "kernels2.cuh"

namespace mgrg {

#ifndef LEAN_TY_F32
#define LEAN_TY_F32 3 // measured: 3 = 2.13 ms, 4 = 2.19 ms at L10 (MINB 3; 4 CTAs/SM spill-free variants are slower)
#endif
#ifndef LEAN_DEC_MINB
#define LEAN_DEC_MINB 3
#endif
// CTAs per SM of the exact-policy instantiations (no FMA contraction: more
// live temporaries), measured (profiles/r2/tuning): decompose f32 4 (3.94 ->
// 3.54 ms at 1025^3 L10), f64 2 (5.23 -> 3.68 ms at 1025^2 x 513 L9); load
// vector f32 3, f64 2 (2.93 -> 2.73 ms); GPK inverse 3
#ifndef LEAN_EXACT_MINB_DEC_F32
#define LEAN_EXACT_MINB_DEC_F32 4
#endif
#ifndef LEAN_EXACT_MINB_DEC_F64
#define LEAN_EXACT_MINB_DEC_F64 2
#endif
#ifndef LEAN_EXACT_MINB_RL_F32
#define LEAN_EXACT_MINB_RL_F32 3
#endif
#ifndef LEAN_EXACT_MINB_RL_F64
#define LEAN_EXACT_MINB_RL_F64 2
#endif
#ifndef LEAN_EXACT_MINB_RG
#define LEAN_EXACT_MINB_RG 3
#endif
#ifndef LEAN_TY_F64
#define LEAN_TY_F64 3 // measured (1025^2 x 513 f64, L9): TY 2 / MINB 3 2.59 ms, 2 / 2 2.33, 3 / 2 1.93, 4 / 2 2.41
#endif
#ifndef LEAN_DEC_MINB_F64
#define LEAN_DEC_MINB_F64 2
#endif
template <typename R> __host__ __device__ constexpr int lean_ty() { return sizeof(R) == 4 ? LEAN_TY_F32 : LEAN_TY_F64; } // coarse y rows per warp band
#ifndef LEAN_ZC_MAX
#define LEAN_ZC_MAX 32
#endif
constexpr int kLeanZC = LEAN_ZC_MAX; // coarse z planes per warp chunk (at most)
constexpr int kLeanWPB = 4;   // warps per CTA (independent tiles)
constexpr int kLeanOut = 30;  // coarse x outputs per warp
#ifndef LEAN_RL_TY
#define LEAN_RL_TY 6
#endif
#ifndef LEAN_RL_MINB
#define LEAN_RL_MINB 3
#endif

// Warp tiles of a lean launch: x tiles of 30 coarse columns, y bands of
// lean_ty<R>() coarse rows, z chunks of kLeanZC coarse planes (1 in 2-D).
struct LeanTiles {
  uint32_t ntx, nty, ntz;
  int zc;           // coarse z planes per chunk (host-chosen per level: enough warps)
  uint32_t tz0 = 0; // first z chunk of this launch (pipelined host path: slab groups)
  __host__ __device__ uint64_t warps() const { return uint64_t(ntx) * nty * ntz; }
};

template <typename R> struct Vec2;
template <> struct Vec2<float> { using T = float2; };
template <> struct Vec2<double> { using T = double2; };

// Per coarse index c of one dimension (padded: entry c+2, zero rows at
// c = -2, -1, m, m+1): the merged R*M weights on taps 2c-2 .. 2c+2 and the
// lerp ratio t of the odd node 2c+1 (0 when it does not exist).  Built on
// the host from the fp64 geometry (mgrg.cu lean_table).
template <typename R> struct LeanW {
  R w[5];
  R t;
  R pad[2];
};

template <typename R> struct W5r {
  R w0, w1, w2, w3, w4;
};
template <typename R> __device__ __forceinline__ W5r<R> lean_w(const LeanW<R> *__restrict__ p) {
  return {__ldg(p->w), __ldg(p->w + 1), __ldg(p->w + 2), __ldg(p->w + 3), __ldg(p->w + 4)};
}

// Arithmetic policy (template FAST): FMA lerps and host-precomputed 5-tap
// FMA stencils, or the exact policy -- the reference's expressions with
// round-to-nearest intrinsics and its merged mass-trans evaluation order
// (stencil_eval<R, false>, kernels2.cuh), bit-identical to the CPU path.
template <typename R, bool FAST> __device__ __forceinline__ R plerp(R a, R b, R t) {
  if constexpr (FAST)
    return fma(t, b - a, a);
  else
    return mgrg::lerp(a, b, t); // a + t * (b - a), kernels.hpp:219
}
template <typename R, bool FAST> __device__ __forceinline__ R psub(R a, R b) {
  if constexpr (FAST)
    return a - b;
  else
    return mgrg::sub(a, b);
}
template <typename R, bool FAST> __device__ __forceinline__ R padd(R a, R b) {
  if constexpr (FAST)
    return a + b;
  else
    return mgrg::add(a, b);
}
template <typename R, bool FAST>
__device__ __forceinline__ R pstencil(const W5r<R> &w, const Stencil<R> &s, R t0, R t1, R t2,
                                      R t3, R t4) {
  if constexpr (FAST) {
    R v = w.w0 * t0;
    v = fma(w.w1, t1, v);
    v = fma(w.w2, t2, v);
    v = fma(w.w3, t3, v);
    return fma(w.w4, t4, v);
  } else {
    return stencil_eval<R, false>(s, t0, t1, t2, t3, t4);
  }
}

// Merged R*M along x for the lane's output column: taps are the vec(C)
// values at 2qc-2 .. 2qc+2 (lane a-1's pair, own pair, lane a+1's even).
template <typename R, bool FAST>
__device__ __forceinline__ R lean_xpass(const W5r<R> &wx, const Stencil<R> &sx, R ce, R co) {
  const R em = __shfl_up_sync(0xffffffffu, ce, 1);
  const R om = __shfl_up_sync(0xffffffffu, co, 1);
  if constexpr (FAST) {
    const R ep = __shfl_down_sync(0xffffffffu, ce, 1);
    return pstencil<R, FAST>(wx, sx, em, om, ce, co, ep);
  } else { // the q+1 term is the next lane's q-1 term (st_ml)
    const R ml = st_ml(sx, em, om, ce);
    const R mr = __shfl_down_sync(0xffffffffu, ml, 1);
    return st_combine(sx, em, om, ce, co, ml, mr);
  }
}
// Same on a row whose even nodes are kept (coarse in every other dim): the
// even taps are zero.
template <typename R, bool FAST>
__device__ __forceinline__ R lean_xpass_odd(const W5r<R> &wx, const Stencil<R> &sx, R co) {
  const R om = __shfl_up_sync(0xffffffffu, co, 1);
  if constexpr (FAST) {
    return fma(wx.w3, co, wx.w1 * om);
  } else {
    const R ml = st_ml(sx, R(0), om, R(0));
    const R mr = __shfl_down_sync(0xffffffffu, ml, 1);
    return st_combine(sx, R(0), om, R(0), co, ml, mr);
  }
}

// Merged R*M along y of the band's x results, output row j (y stencil row
// cy0 + j; rows past the level are clamped -- their outputs are not stored)
// All TY outputs of the band; the exact policy carries output j's q+1 term
// as output j+1's q-1 term (st_ml / st_mr), one stencil live at a time.
template <typename R, bool FAST, int TY>
__device__ __forceinline__ void lean_ypass_all(const W5r<R> *wy, const Stencil<R> *__restrict__ sy,
                                               int cy0, int m1, const R *X, R *Y) {
  if constexpr (FAST) {
#pragma unroll
    for (int j = 0; j < TY; ++j)
      Y[j] = pstencil<R, true>(wy[j], Stencil<R>{}, X[2 * j], X[2 * j + 1], X[2 * j + 2],
                               X[2 * j + 3], X[2 * j + 4]);
  } else {
    R ml = R(0);
#pragma unroll
    for (int j = 0; j < TY; ++j) {
      const Stencil<R> s = sy[min(cy0 + j, m1 - 1)];
      if (j == 0)
        ml = st_ml(s, X[0], X[1], X[2]);
      const R mr = st_mr(s, X[2 * j + 2], X[2 * j + 3], X[2 * j + 4]);
      Y[j] = st_combine(s, X[2 * j], X[2 * j + 1], X[2 * j + 2], X[2 * j + 3], ml, mr);
      ml = mr;
    }
  }
}

template <typename R, bool FAST>
__device__ __forceinline__ R lean_ypass(const W5r<R> *wy, const Stencil<R> *__restrict__ sy,
                                        int row, const R *X, int j) {
  Stencil<R> s;
  if constexpr (!FAST)
    s = sy[row];
  return pstencil<R, FAST>(FAST ? wy[j] : W5r<R>{}, s, X[2 * j], X[2 * j + 1], X[2 * j + 2],
                           X[2 * j + 3], X[2 * j + 4]);
}

template <typename R> __device__ __forceinline__ R flerp(R a, R b, R t) {
  return fma(t, b - a, a);
}

// Paired (even, odd) node updates.  FAST f32: Blackwell's packed FP32x2
// instructions (FADD2 / FFMA2) do both lanes of the pair in one issue slot;
// each component is the same round-to-nearest operation as the scalar FAST
// code, so results are bit-identical to plerp / psub per component.  (Not
// used for the exact policy: ptxas fuses a packed multiply and add into
// FFMA2 even for .rn operations, which would break bit-identity.)
template <typename R, bool FAST>
__device__ __forceinline__ typename Vec2<R>::T plerp2(typename Vec2<R>::T a,
                                                      typename Vec2<R>::T b, R t) {
  if constexpr (FAST && sizeof(R) == 4) {
    return __ffma2_rn(make_float2(t, t), __fadd2_rn(b, make_float2(-a.x, -a.y)), a);
  } else {
    typename Vec2<R>::T r;
    r.x = plerp<R, FAST>(a.x, b.x, t);
    r.y = plerp<R, FAST>(a.y, b.y, t);
    return r;
  }
}
template <typename R, bool FAST>
__device__ __forceinline__ typename Vec2<R>::T psub2(typename Vec2<R>::T a,
                                                     typename Vec2<R>::T b) {
  if constexpr (FAST && sizeof(R) == 4) {
    return __fadd2_rn(a, make_float2(-b.x, -b.y));
  } else {
    typename Vec2<R>::T r;
    r.x = psub<R, FAST>(a.x, b.x);
    r.y = psub<R, FAST>(a.y, b.y);
    return r;
  }
}

template <typename R, bool ALIGNED>
__device__ __forceinline__ Pair<R> lean_pair(const typename Vec2<R>::T &v) {
  if constexpr (ALIGNED)
    return {v.x, v.y};
  else
    return {v.y, __shfl_down_sync(0xffffffffu, v.x, 1)};
}

// Per-warp staging ring of the decompose kernel: 3 plane slots of NR rows;
// a staged row is the 16-byte aligned superset of the lane pairs' 64
// elements (RP elements, NCH 16-byte chunks), fetched with LDGSTS.128 so
// that two planes of loads are in flight while one is processed, without
// holding registers.
template <typename R> struct LeanStage {
  static constexpr int V = 16 / int(sizeof(R));
  static constexpr int NCH = (64 + 2 * V - 2) / V; // ceil((64 + V - 1) / V)
  static constexpr int RP = NCH * V;
};

// Issue the copies of one plane into `slot`.  `pb` points at the plane's
// element 0, q = (element index of pb) mod V, row r starts at element
// rowoff[r] of the plane.  Interior planes (every chunk inside the array)
// take the unchecked path; near the array ends chunks before element 0 are
// skipped (invalid columns) and chunks crossing the end go element-wise.
template <typename R, int NR>
__device__ __forceinline__ void lean_stage_plane(R *slot, const R *__restrict__ in,
                                                 const R *__restrict__ pb, int q,
                                                 const int *rowoff, bool interior,
                                                 int64_t pbase, int64_t ntot, int lane) {
  constexpr int V = LeanStage<R>::V, NCH = LeanStage<R>::NCH, RP = LeanStage<R>::RP;
  // lane c copies chunk c (and c + 32 when NCH > 32) of every row
  R *sl = slot + lane * V;
  if (interior) {
    // 32-bit element indices (lean plans have N < 2^32): chunk c of row r
    // starts at ((pbase + rowoff[r]) & ~(V-1)) + c*V = (pbase + rowoff[r] +
    // c*V) & ~(V-1) -- one add, one mask and one wide multiply-add per copy
    const uint32_t pl = uint32_t(pbase) + uint32_t(lane * V);
    if (lane < NCH) {
#pragma unroll
      for (int r = 0; r < NR; ++r)
        cp_async16(sl + r * RP, in + ((pl + uint32_t(rowoff[r])) & ~uint32_t(V - 1)));
    }
    if (NCH > 32 && lane + 32 < NCH) {
#pragma unroll
      for (int r = 0; r < NR; ++r)
        cp_async16(sl + r * RP + 32 * V,
                   in + ((pl + uint32_t(rowoff[r] + 32 * V)) & ~uint32_t(V - 1)));
    }
    return;
  }
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int s0 = ((q + rowoff[r]) & ~(V - 1)) - q;
#pragma unroll
    for (int c = lane; c < NCH; c += 32) {
      const int64_t g = pbase + s0 + int64_t(c) * V;
      R *d = slot + r * RP + c * V;
      if (g >= 0 && g + V <= ntot) {
        cp_async16(d, pb + s0 + c * V);
      } else if (g >= 0) {
#pragma unroll
        for (int v = 0; v < V; ++v)
          if (g + v < ntot)
            cp_async(d + v, pb + s0 + c * V + v);
      }
    }
  }
}

// Class/packed stores of one plane as 32-bit element indices (lean plans
// have N < 2^32; indices may wrap below zero for masked rows): row r of the
// band writes its even node to (r even: pe0, else cls)[ie[r&1] + ex_e*(r>>1)]
// and its odd node to cls[io[r&1] + ex_o*(r>>1)].
template <typename R> struct PlaneOut {
  R *pe0;                     // even rows' even nodes: P (even plane) or cls
  uint32_t ie0, io0, ie1, io1; // even rows (e, o), odd rows (e, o)
};

// ---------------------------------------------------------------------------
// One fine plane of the band: loads, GPK (interpolant W from the in-plane
// prolongation, or from the z lerp of the two even planes around), class
// stores, x pass and y pass.  EVEN: plane is coarse along z.
//   PAR: parity of the plane's row 0 (aligned rows are those with
//        (r + PAR) even, r = band row index, band row 0 even).
template <typename R, int TY, bool EVEN, bool FAST>
__device__ __forceinline__ void lean_plane(
    const R *__restrict__ slot, int q, const int *rowoff, R txr, const R *tyr,
    const W5r<R> &wx, const W5r<R> *wy, const Stencil<R> &sx,
    const Stencil<R> *__restrict__ sy, int cy0, int m1, bool ve, bool vo, uint32_t stmask_e,
    uint32_t stmask_o, const PlaneOut<R> &po, R *__restrict__ cls, int ex_e, int ex_o,
    typename Vec2<R>::T *W, const typename Vec2<R>::T *WL, R tz, R *Y) {
  constexpr int NR = 2 * TY + 3;
  constexpr int RP = LeanStage<R>::RP;
  using V = typename Vec2<R>::T;
  const int lane = threadIdx.x & 31;
  V raw[NR];
  // staged row r holds the band row from its 16-byte aligned start; the
  // lane's even node sits at shift_r + 2*lane, shift_r = (q + rowoff[r]) mod
  // V.  EVEN planes: aligned rows (even shift) are the even ones; odd
  // planes: the odd ones.
  const R *sl = slot + 2 * lane;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const R *p = sl + r * RP + ((q + rowoff[r]) & (LeanStage<R>::V - 1));
    if (((r & 1) == 0) == EVEN)
      raw[r] = *reinterpret_cast<const V *>(p);
    else
      raw[r] = *reinterpret_cast<const V *>(p - 1);
  }
  // u[r] = (even node, odd node) of the lane's pair on band row r
  V u[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    if (((r & 1) == 0) == EVEN) {
      u[r] = raw[r];
    } else {
      u[r].x = raw[r].y;
      u[r].y = __shfl_down_sync(0xffffffffu, raw[r].x, 1);
    }
  }
  R X[NR];
  if constexpr (EVEN) {
#pragma unroll
    for (int r = 0; r < NR; r += 2) {
      const R un = __shfl_down_sync(0xffffffffu, u[r].x, 1);
      W[r].x = u[r].x;
      W[r].y = plerp<R, FAST>(u[r].x, un, txr);
    }
#pragma unroll
    for (int r = 1; r < NR; r += 2)
      W[r] = plerp2<R, FAST>(W[r - 1], W[r + 1], tyr[r >> 1]);
  }
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    V w;
    if constexpr (EVEN)
      w = W[r];
    else
      w = plerp2<R, FAST>(WL[r], W[r], tz);
    const V c = psub2<R, FAST>(u[r], w);
    const bool kept = EVEN && !(r & 1); // even node coarse in every dim
    const R ce = (kept || !ve) ? R(0) : c.x;
    const R co = vo ? c.y : R(0);
    const int rr = r >> 1;
    if ((stmask_e >> r) & 1u)
      ((r & 1) ? cls : po.pe0)[((r & 1) ? po.ie1 : po.ie0) + uint32_t(ex_e * rr)] =
          kept ? u[r].x : ce;
    if ((stmask_o >> r) & 1u)
      cls[((r & 1) ? po.io1 : po.io0) + uint32_t(ex_o * rr)] = co;
    X[r] = kept ? lean_xpass_odd<R, FAST>(wx, sx, co) : lean_xpass<R, FAST>(wx, sx, ce, co);
  }
  lean_ypass_all<R, FAST, TY>(wy, sy, cy0, m1, X, Y);
}

// ---------------------------------------------------------------------------
// Decompose level kernel: GPK forward (class stores, packed kept nodes) and
// the load vector f = (R*M)_z (R*M)_y (R*M)_x vec(C) on the coarse lattice.
// Z3 = false: 2-D level (n2 == 1), one plane.
template <typename R> __host__ __device__ constexpr size_t lean_dec_smem() {
  return size_t(kLeanWPB) * 3 * (2 * lean_ty<R>() + 3) * LeanStage<R>::RP * sizeof(R);
}

template <typename R, bool Z3, bool FAST>
__global__ void __launch_bounds__(32 * kLeanWPB, !FAST ? (sizeof(R) == 4 ? LEAN_EXACT_MINB_DEC_F32 : LEAN_EXACT_MINB_DEC_F64) : (sizeof(R) == 4 ? LEAN_DEC_MINB : LEAN_DEC_MINB_F64))
    lean_dec_kernel(LevelGeom<R> g, const LeanW<R> *__restrict__ lx,
                    const LeanW<R> *__restrict__ ly, const LeanW<R> *__restrict__ lz,
                    const Stencil<R> *__restrict__ sxt, const Stencil<R> *__restrict__ syt,
                    const Stencil<R> *__restrict__ szt, const R *__restrict__ in,
                    R *__restrict__ cls, R *__restrict__ P, R *__restrict__ f, LeanTiles tl) {
  pdl_wait();
  constexpr int TY = lean_ty<R>(), NR = 2 * TY + 3;
  constexpr int V = LeanStage<R>::V, SLOT = NR * LeanStage<R>::RP;
  extern __shared__ __align__(16) unsigned char lean_raw_sm[];
  const int lane = threadIdx.x & 31;
  R *ring = reinterpret_cast<R *>(lean_raw_sm) + size_t(threadIdx.x >> 5) * 3 * SLOT;
  const uint64_t wid = uint64_t(blockIdx.x) * kLeanWPB + (threadIdx.x >> 5);
  if (wid >= tl.warps())
    return;
  const uint32_t tx = uint32_t(wid % tl.ntx);
  const uint64_t rest = wid / tl.ntx;
  const uint32_t tyb = uint32_t(rest % tl.nty), tzc = uint32_t(rest / tl.nty) + tl.tz0;

  const int n0 = int(g.n[0]), n1 = int(g.n[1]), n2 = int(g.n[2]);
  const int m0 = int(g.m[0]), m1 = int(g.m[1]), m2 = int(g.m[2]);
  const int64_t nxy = int64_t(n0) * n1, ntot = nxy * n2;

  // ---- lane x geometry
  const int qc = int(kLeanOut * tx) - 1 + lane;
  const bool ve = qc >= 0 && qc < m0;     // even node 2qc exists
  const bool vo = qc >= 0 && qc + 1 < m0; // odd node 2qc+1 exists
  const bool outl = lane >= 1 && lane <= kLeanOut && ve;
  const LeanW<R> *lxq = lx + (min(max(qc, -2), m0 + 1) + 2);
  const R txr = __ldg(&lxq->t);
  W5r<R> wx = lean_w(lxq);
  if (!outl)
    wx = {R(0), R(0), R(0), R(0), R(0)};
  Stencil<R> sx{}; // exact policy: the lane's x stencil (non-output lanes: unused)
  if constexpr (!FAST)
    sx = sxt[min(max(qc, 0), m0 - 1)];
  const int X0 = 2 * (int(kLeanOut * tx) - 1); // lane 0's even node

  // ---- y band: rows Y0 + r, r = 0 .. NR-1
  const int cy0 = int(tyb) * TY, cy1 = min(cy0 + TY, m1);
  const int Y0 = 2 * cy0 - 2;
  int rowoff[NR]; // within-plane element offset of band row r (n0 * n1 < 2^31)
  uint32_t ownrows = 0;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int y = Y0 + r;
    const bool rv = y >= 0 && y < n1;
    // invalid rows stage a row of the same parity (values unused: weights 0)
    rowoff[r] = (rv ? y : (r & 1)) * n0 + X0;
    if (rv && r >= 2 && r < 2 + 2 * (cy1 - cy0))
      ownrows |= 1u << r;
  }
  R tyr[TY + 1];
#pragma unroll
  for (int i = 0; i <= TY; ++i)
    tyr[i] = __ldg(&ly[min(cy0 - 1 + i, m1 + 1) + 2].t); // odd row 2(cy0 - 1 + i) + 1
  W5r<R> wy[TY];
#pragma unroll
  for (int j = 0; j < TY; ++j)
    wy[j] = lean_w(ly + min(cy0 + j, m1 + 1) + 2);
  const uint32_t st_e = outl ? ownrows : 0u, st_o = (outl && vo) ? ownrows : 0u;

  // ---- z chunk and the plane sequence: j = 0: even plane 2(cz0-1); then
  // per step k = cz0 .. cz1: even plane 2k (j odd), odd plane 2k-1 (j even)
  const int cz0 = Z3 ? int(tzc) * tl.zc : 0;
  const int cz1 = Z3 ? min(cz0 + tl.zc, m2) : 1;
  const int kbeg = Z3 ? cz0 - 1 : 0, kend = Z3 ? cz1 : 0;
  const int J = Z3 ? 2 * (cz1 - cz0 + 1) + 1 : 1;
  auto plane_of = [&](int j) -> int { // fine plane index, or -1 when skipped
    if (!Z3)
      return 0;
    const int k = j == 0 ? cz0 - 1 : cz0 + (j - 1) / 2;
    const int p = (j == 0 || (j & 1)) ? 2 * k : 2 * k - 1;
    const bool ok = (j & 1) || j == 0 ? (p >= 0 && p < n2) : (p >= 1 && p < n2);
    return ok ? p : -1;
  };
  // rows of the band lie in [rowoff[0], rowoff[NR-1] + 64 + V) of a plane
  int rlo = rowoff[0], rhi = rowoff[0];
#pragma unroll
  for (int r = 1; r < NR; ++r) {
    rlo = min(rlo, rowoff[r]);
    rhi = max(rhi, rowoff[r]);
  }
  rlo -= V;
  rhi += LeanStage<R>::RP + V;
  auto issue = [&](int j) {
    const int p = j < J ? plane_of(j) : -1;
    if (p >= 0) {
      const int64_t pbase = int64_t(p) * nxy;
      const bool interior = pbase + rlo >= 0 && pbase + rhi <= ntot;
      const int slot = j % 3;
      lean_stage_plane<R, NR>(ring + slot * SLOT, in, in + pbase, int(pbase & (V - 1)),
                              rowoff, interior, pbase, ntot, lane);
    }
    cp_async_commit();
  };
  auto q_of = [&](int p) -> int { return int((int64_t(p) * nxy) & (V - 1)); };

  using V2 = typename Vec2<R>::T;
  V2 WL[NR]; // the previous even plane's interpolant (even, odd node)
#pragma unroll
  for (int r = 0; r < NR; ++r)
    WL[r].x = WL[r].y = R(0);
  R accM[TY], acc0[TY]; // FAST: partial f of outputs k-1 and k at step k
  R YEm2[TY], YOm1[TY], YEm1[TY]; // exact: carried q-1 term; y results of planes 2k-3, 2k-2
#pragma unroll
  for (int j = 0; j < TY; ++j)
    accM[j] = acc0[j] = YEm2[j] = YOm1[j] = YEm1[j] = R(0);
  const int64_t m01 = int64_t(m0) * m1;
  const uint32_t fq0 = uint32_t(qc + m0 * cy0); // f index of output row cy0 (may wrap: masked)

  issue(0);
  issue(1);
  int j = 0, js = 0; // plane counter and its ring slot (j % 3)
  for (int k = kbeg; k <= kend; ++k) {
    R YE[TY], YO[TY];
    V2 W[NR];
    // ================= even plane 2k =================
    {
      const int pe = 2 * k;
      issue(j + 2);
      cp_async_wait<2>();
      __syncwarp();
      if (pe >= 0 && pe < n2) {
        const bool own = pe >= 2 * cz0 && pe < 2 * cz1;
        const int64_t yb = int64_t(cy0) - 1; // rank of band row 0
        PlaneOut<R> po;
        po.pe0 = P;
        po.ie0 = uint32_t(qc + int64_t(m0) * (yb + int64_t(m1) * k));
        po.io0 = uint32_t(g.tbase[1] + qc + int64_t(m0 - 1) * (yb + int64_t(m1) * k));
        po.ie1 = uint32_t(g.tbase[2] + qc + int64_t(m0) * (yb + int64_t(m1 - 1) * k));
        po.io1 = uint32_t(g.tbase[3] + qc + int64_t(m0 - 1) * (yb + int64_t(m1 - 1) * k));
        lean_plane<R, TY, true, FAST>(ring + js * SLOT, q_of(pe), rowoff, txr, tyr, wx, wy, sx,
                                      syt, cy0, m1, ve,
                                vo, own ? st_e : 0u, own ? st_o : 0u, po, cls, m0, m0 - 1, W,
                                nullptr, R(0), YE);
      } else {
#pragma unroll
        for (int r = 0; r < NR; ++r)
          W[r].x = W[r].y = R(0);
#pragma unroll
        for (int i = 0; i < TY; ++i)
          YE[i] = R(0);
      }
      __syncwarp(); // slot j % 3 is refilled by issue(j + 3)
      ++j;
      js = js == 2 ? 0 : js + 1;
    }
    if constexpr (!Z3) {
#pragma unroll
      for (int i = 0; i < TY; ++i)
        if (outl && cy0 + i < cy1)
          f[fq0 + uint32_t(m0 * i)] = YE[i];
      break;
    }
    // ================= odd plane 2k - 1 =================
    const int pz = 2 * k - 1;
    const LeanW<R> *lzk = lz + k + 1; // coarse c = k - 1 (padded index c + 2)
    if (k >= cz0) {
      issue(j + 2);
      cp_async_wait<2>();
      __syncwarp();
      if (pz >= 1 && pz < n2) {
        const bool own = pz >= 2 * cz0 && pz < 2 * cz1;
        const int64_t yb = int64_t(cy0) - 1;
        const int64_t zr = k - 1;
        PlaneOut<R> po;
        po.pe0 = cls;
        po.ie0 = uint32_t(g.tbase[4] + qc + int64_t(m0) * (yb + int64_t(m1) * zr));
        po.io0 = uint32_t(g.tbase[5] + qc + int64_t(m0 - 1) * (yb + int64_t(m1) * zr));
        po.ie1 = uint32_t(g.tbase[6] + qc + int64_t(m0) * (yb + int64_t(m1 - 1) * zr));
        po.io1 = uint32_t(g.tbase[7] + qc + int64_t(m0 - 1) * (yb + int64_t(m1 - 1) * zr));
        lean_plane<R, TY, false, FAST>(ring + js * SLOT, q_of(pz), rowoff, txr, tyr, wx, wy, sx,
                                       syt, cy0, m1, ve,
                                 vo, own ? st_e : 0u, own ? st_o : 0u, po, cls, m0, m0 - 1, W,
                                 WL, __ldg(&lzk->t), YO);
      } else {
#pragma unroll
        for (int i = 0; i < TY; ++i)
          YO[i] = R(0);
      }
      __syncwarp();
      ++j;
      js = js == 2 ? 0 : js + 1;
    } else {
#pragma unroll
      for (int i = 0; i < TY; ++i)
        YO[i] = R(0);
    }
#pragma unroll
    for (int r = 0; r < NR; ++r)
      WL[r] = W[r];
    // ================= z pass =================
    const bool emit = outl && k - 1 >= cz0 && k - 1 < cz1;
    if constexpr (FAST) { // rolling accumulators
      const R a3 = __ldg(lzk->w + 3), a4 = __ldg(lzk->w + 4);     // output k-1
      const R b1 = __ldg(lzk[1].w + 1), b2 = __ldg(lzk[1].w + 2); // output k
      const R c0 = __ldg(lzk[2].w);                               // output k+1
#pragma unroll
      for (int i = 0; i < TY; ++i) {
        const R out = fma(a3, YO[i], fma(a4, YE[i], accM[i]));
        if (emit && cy0 + i < cy1)
          f[fq0 + uint32_t(m0 * i) + uint32_t(m01) * uint32_t(k - 1)] = out;
        accM[i] = fma(b1, YO[i], fma(b2, YE[i], acc0[i]));
        acc0[i] = c0 * YE[i];
      }
    } else { // exact: output k-1 from planes 2k-3 .. 2k; its q-1 term is
      // output k-2's q+1 term, carried in YEm2 (st_ml / st_mr; computed from
      // step cz0 on, where output cz0-1's q+1 term is output cz0's q-1 term)
      const bool need = k >= 1 && k >= cz0 && k - 1 < cz1;
      Stencil<R> sk{};
      if (need)
        sk = szt[k - 1];
#pragma unroll
      for (int i = 0; i < TY; ++i) {
        const R mr = st_mr(sk, YEm1[i], YO[i], YE[i]);
        if (emit && cy0 + i < cy1)
          f[fq0 + uint32_t(m0 * i) + uint32_t(m01) * uint32_t(k - 1)] =
              st_combine(sk, R(0), YOm1[i], YEm1[i], YO[i], YEm2[i], mr);
        YEm2[i] = mr;
        YOm1[i] = YO[i];
        YEm1[i] = YE[i];
      }
    }
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// Recompose load vector: f = (R*M)_z (R*M)_y (R*M)_x vec(C) read from the
// class buffer of level l (coarse-in-every-dim nodes are zero).  Same warp
// tiling and band walk as lean_dec_kernel; the class rows are coalesced
// 4/8-byte loads (lane qc of a type row is element qc).
#ifndef LEAN_RL_TY_F64
#define LEAN_RL_TY_F64 4
#endif
#ifndef LEAN_RL_MINB_F64
#define LEAN_RL_MINB_F64 2 // measured (1025^2 x 513 f64, L9): MINB 3 (168 regs, spills) 1.13 ms, 2 (246) 1.07
#endif
#ifndef LEAN_RL_TY_EXACT
#define LEAN_RL_TY_EXACT 5 // exact f32 at 1025^3 L10: TY 6 3.41 ms (spills), 5 2.74, 4 2.82, 3 3.02
#endif
template <typename R, bool FAST = true> __host__ __device__ constexpr int lean_ty_rl() {
  // taller band: fewer halo rows (no W registers here); the exact policy's
  // unfused stencils keep more temporaries live
  return sizeof(R) == 4 ? (FAST ? LEAN_RL_TY : LEAN_RL_TY_EXACT) : LEAN_RL_TY_F64;
}

template <typename R, bool Z3, bool FAST>
__global__ void __launch_bounds__(32 * kLeanWPB, !FAST ? (sizeof(R) == 4 ? LEAN_EXACT_MINB_RL_F32 : LEAN_EXACT_MINB_RL_F64) : (sizeof(R) == 4 ? LEAN_RL_MINB : LEAN_RL_MINB_F64))
    lean_rload_kernel(LevelGeom<R> g, const LeanW<R> *__restrict__ lx,
                      const LeanW<R> *__restrict__ ly, const LeanW<R> *__restrict__ lz,
                      const Stencil<R> *__restrict__ sxt, const Stencil<R> *__restrict__ syt,
                      const Stencil<R> *__restrict__ szt, const R *__restrict__ cls,
                      R *__restrict__ f, LeanTiles tl) {
  pdl_wait();
  constexpr int TY = lean_ty_rl<R, FAST>(), NR = 2 * TY + 3;
  const int lane = threadIdx.x & 31;
  const uint64_t wid = uint64_t(blockIdx.x) * kLeanWPB + (threadIdx.x >> 5);
  if (wid >= tl.warps())
    return;
  const uint32_t tx = uint32_t(wid % tl.ntx);
  const uint64_t rest = wid / tl.ntx;
  const uint32_t tyb = uint32_t(rest % tl.nty), tzc = uint32_t(rest / tl.nty) + tl.tz0;
  const int n1 = int(g.n[1]), n2 = int(g.n[2]);
  const int m0 = int(g.m[0]), m1 = int(g.m[1]), m2 = int(g.m[2]);

  const int qc = int(kLeanOut * tx) - 1 + lane;
  const bool ve = qc >= 0 && qc < m0;
  const bool vo = qc >= 0 && qc + 1 < m0;
  const bool outl = lane >= 1 && lane <= kLeanOut && ve;
  W5r<R> wx = lean_w(lx + (min(max(qc, -2), m0 + 1) + 2));
  if (!outl)
    wx = {R(0), R(0), R(0), R(0), R(0)};
  Stencil<R> sx{}; // exact policy: the lane's x stencil
  if constexpr (!FAST)
    sx = sxt[min(max(qc, 0), m0 - 1)];
  const int qe = min(max(qc, 0), m0 - 1), qo = min(max(qc, 0), max(m0 - 2, 0));

  const int cy0 = int(tyb) * TY, cy1 = min(cy0 + TY, m1);
  const int Y0 = 2 * cy0 - 2;
  uint32_t rowvalid = 0;
#pragma unroll
  for (int r = 0; r < NR; ++r)
    if (Y0 + r >= 0 && Y0 + r < n1)
      rowvalid |= 1u << r;
  W5r<R> wy[TY];
#pragma unroll
  for (int j = 0; j < TY; ++j)
    wy[j] = lean_w(ly + min(cy0 + j, m1 + 1) + 2);
  // class row rank of band row r is cy0 - 1 + (r >> 1); ranks outside the
  // type's y range belong to invalid rows (masked) and read a valid row
  const int yrmax_e = m1 - 1, yrmax_o = m1 - 2;

  const int cz0 = Z3 ? int(tzc) * tl.zc : 0;
  const int cz1 = Z3 ? min(cz0 + tl.zc, m2) : 1;
  R accM[TY], acc0[TY];          // FAST: partial f of outputs k-1 and k
  R YEm2[TY], YOm1[TY], YEm1[TY]; // exact: carried q-1 term; y results of planes 2k-3, 2k-2
#pragma unroll
  for (int j = 0; j < TY; ++j)
    accM[j] = acc0[j] = YEm2[j] = YOm1[j] = YEm1[j] = R(0);
  const int64_t m01 = int64_t(m0) * m1;
  const uint32_t fq0 = uint32_t(qc + m0 * cy0); // f index of output row cy0 (may wrap: masked)

  // class row offsets of band row r (rank cy0 - 1 + (r >> 1) clamped into
  // the type's y range; invalid rows are masked), loop invariant
  uint32_t oe[NR], oo[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const uint32_t rk =
        uint32_t(min(max(cy0 - 1 + (r >> 1), 0), (r & 1) ? max(yrmax_o, 0) : yrmax_e));
    oe[r] = uint32_t(m0) * rk;
    oo[r] = uint32_t(m0 - 1) * rk;
  }

  for (int k = Z3 ? cz0 - 1 : 0; k <= (Z3 ? cz1 : 0); ++k) {
    R YE[TY], YO[TY];
    const int pe = 2 * k, pz = pe - 1;
    const bool ev = pe >= 0 && pe < n2;
    const bool ov = Z3 && k >= cz0 && pz >= 1 && pz < n2;
    // ---- both planes' loads first (one batch of independent loads per
    // step); invalid planes read a valid one and are zeroed below
    // 32-bit element indices into the class buffer (lean plans: N < 2^32)
    const uint32_t ke = ev ? uint32_t(k) : 0u, ko = ov ? uint32_t(k - 1) : 0u;
    const uint32_t b1 = qo + uint32_t(g.tbase[1]) + uint32_t(m0 - 1) * (uint32_t(m1) * ke);
    const uint32_t b2 = qe + uint32_t(g.tbase[2]) + uint32_t(m0) * (uint32_t(m1 - 1) * ke);
    const uint32_t b3 = qo + uint32_t(g.tbase[3]) + uint32_t(m0 - 1) * (uint32_t(m1 - 1) * ke);
    R ueE[NR], uoE[NR], ueO[NR], uoO[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      ueE[r] = (r & 1) ? __ldg(cls + (b2 + oe[r])) : R(0); // even rows: kept nodes
      uoE[r] = __ldg(cls + (((r & 1) ? b3 : b1) + oo[r]));
    }
    if constexpr (Z3) {
      const uint32_t b4 = qe + uint32_t(g.tbase[4]) + uint32_t(m0) * (uint32_t(m1) * ko);
      const uint32_t b5 = qo + uint32_t(g.tbase[5]) + uint32_t(m0 - 1) * (uint32_t(m1) * ko);
      const uint32_t b6 = qe + uint32_t(g.tbase[6]) + uint32_t(m0) * (uint32_t(m1 - 1) * ko);
      const uint32_t b7 =
          qo + uint32_t(g.tbase[7]) + uint32_t(m0 - 1) * (uint32_t(m1 - 1) * ko);
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        ueO[r] = __ldg(cls + (((r & 1) ? b6 : b4) + oe[r]));
        uoO[r] = __ldg(cls + (((r & 1) ? b7 : b5) + oo[r]));
      }
    }
    // ---- even plane
    {
      R X[NR];
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const bool rv = ev && ((rowvalid >> r) & 1u);
        const R co = (vo && rv) ? uoE[r] : R(0);
        if (!(r & 1)) {
          X[r] = lean_xpass_odd<R, FAST>(wx, sx, co);
        } else {
          const R ce = (ve && rv) ? ueE[r] : R(0);
          X[r] = lean_xpass<R, FAST>(wx, sx, ce, co);
        }
      }
      lean_ypass_all<R, FAST, TY>(wy, syt, cy0, m1, X, YE);
    }
    if constexpr (!Z3) {
#pragma unroll
      for (int j = 0; j < TY; ++j)
        if (outl && cy0 + j < cy1)
          f[fq0 + uint32_t(m0 * j)] = YE[j];
      break;
    }
    const LeanW<R> *lzk = lz + k + 1;
    // ---- odd plane
    {
      R X[NR];
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const bool rv = ov && ((rowvalid >> r) & 1u);
        const R ce = (ve && rv) ? ueO[r] : R(0);
        const R co = (vo && rv) ? uoO[r] : R(0);
        X[r] = lean_xpass<R, FAST>(wx, sx, ce, co);
      }
      lean_ypass_all<R, FAST, TY>(wy, syt, cy0, m1, X, YO);
    }
    const bool emit = outl && k - 1 >= cz0 && k - 1 < cz1;
    if constexpr (FAST) {
      const R a3 = __ldg(lzk->w + 3), a4 = __ldg(lzk->w + 4);
      const R b1 = __ldg(lzk[1].w + 1), b2 = __ldg(lzk[1].w + 2);
      const R c0 = __ldg(lzk[2].w);
#pragma unroll
      for (int j = 0; j < TY; ++j) {
        const R out = fma(a3, YO[j], fma(a4, YE[j], accM[j]));
        if (emit && cy0 + j < cy1)
          f[fq0 + uint32_t(m0 * j) + uint32_t(m01) * uint32_t(k - 1)] = out;
        accM[j] = fma(b1, YO[j], fma(b2, YE[j], acc0[j]));
        acc0[j] = c0 * YE[j];
      }
    } else { // exact: as in lean_dec_kernel (q-1 term carried in YEm2)
      const bool need = k >= 1 && k >= cz0 && k - 1 < cz1;
      Stencil<R> sk{};
      if (need)
        sk = szt[k - 1];
#pragma unroll
      for (int j = 0; j < TY; ++j) {
        const R mr = st_mr(sk, YEm1[j], YO[j], YE[j]);
        if (emit && cy0 + j < cy1)
          f[fq0 + uint32_t(m0 * j) + uint32_t(m01) * uint32_t(k - 1)] =
              st_combine(sk, R(0), YOm1[j], YEm1[j], YO[j], YEm2[j], mr);
        YEm2[j] = mr;
        YOm1[j] = YO[j];
        YEm1[j] = YE[j];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Recompose GPK inverse: level array = prolongation of the corrected coarse
// lattice (x -> y -> z lerps) + the class values at fine nodes.  Lane a of
// a warp owns coarse column qc = 31*tx + a (lane 31 is the x-lerp halo),
// the warp a band of TG coarse rows (fine rows 2cy0 .. 2cy1-1, plus the
// coarse row cy1 for the last odd row) through a chunk of coarse planes;
// the interpolant of the previous even plane is carried in registers.
// CLS = false: classes above classes_used (all zero): pure prolongation.
#ifndef LEAN_RG_TG
#define LEAN_RG_TG 3 // measured with LEAN_RG_PF=1: TG 2 / 3 / 4 = 1.90 / 1.75 / 1.92 ms at L10
#endif
#ifndef LEAN_RG_MINB
#define LEAN_RG_MINB 3 // with TG 3 + prefetch: 3 (143 regs) 1.72 ms, 4 (128) 1.76, 5 (96) 2.46
#endif
#ifndef LEAN_RG_PF
#define LEAN_RG_PF 1 // the loads of step k+1 are issued before step k computes
#endif
#ifndef LEAN_RG_TG_F64
#define LEAN_RG_TG_F64 2
#endif
#ifndef LEAN_RG_MINB_F64
#define LEAN_RG_MINB_F64 LEAN_RG_MINB
#endif
template <typename R> __host__ __device__ constexpr int lean_tg() {
  return sizeof(R) == 4 ? LEAN_RG_TG : LEAN_RG_TG_F64;
}
constexpr int kLeanGOut = 31;

template <typename R, bool ALIGNED>
__device__ __forceinline__ void lean_store_pair(R *p, R e, R o, bool we, bool wo) {
  // p points at the lane's even node
  if constexpr (ALIGNED) {
    if (we && wo) {
      using V = typename Vec2<R>::T;
      V v;
      v.x = e;
      v.y = o;
      *reinterpret_cast<V *>(p) = v;
      return;
    }
  }
  if (we)
    p[0] = e;
  if (wo)
    p[1] = o;
}

template <typename R, bool Z3, bool CLS, bool FAST>
__global__ void __launch_bounds__(32 * kLeanWPB, !FAST ? LEAN_EXACT_MINB_RG : (sizeof(R) == 4 ? LEAN_RG_MINB : LEAN_RG_MINB_F64))
    lean_rgpk_kernel(LevelGeom<R> g, const LeanW<R> *__restrict__ lx,
                     const LeanW<R> *__restrict__ ly, const LeanW<R> *__restrict__ lz,
                     const R *__restrict__ coarse, const R *__restrict__ cls,
                     R *__restrict__ out, LeanTiles tl) {
  pdl_wait();
  constexpr int TG = lean_tg<R>(), NF = 2 * TG + 1; // fine rows incl. halo row 2cy1
  const int lane = threadIdx.x & 31;
  const uint64_t wid = uint64_t(blockIdx.x) * kLeanWPB + (threadIdx.x >> 5);
  if (wid >= tl.warps())
    return;
  const uint32_t tx = uint32_t(wid % tl.ntx);
  const uint64_t rest = wid / tl.ntx;
  const uint32_t tyb = uint32_t(rest % tl.nty), tzc = uint32_t(rest / tl.nty) + tl.tz0;
  const int n0 = int(g.n[0]), n1 = int(g.n[1]), n2 = int(g.n[2]);
  const int m0 = int(g.m[0]), m1 = int(g.m[1]), m2 = int(g.m[2]);
  const int64_t nxy = int64_t(n0) * n1;
  const int64_t m01 = int64_t(m0) * m1;

  const int qc = int(kLeanGOut * tx) + lane;
  const bool own = lane < kLeanGOut && qc < m0; // writes e (and o if it exists)
  const bool ownO = own && qc + 1 < m0;
  const int qe = min(qc, m0 - 1), qo = min(qc, max(m0 - 2, 0));
  const R txr = __ldg(&lx[min(qc, m0 + 1) + 2].t);

  const int cy0 = int(tyb) * TG, cy1 = min(cy0 + TG, m1);
  // fine rows 2cy0 + i, i = 0 .. 2TG (i = 2TG: halo, never written)
  uint32_t wrow = 0;
#pragma unroll
  for (int i = 0; i < 2 * TG; ++i)
    if (2 * cy0 + i < n1 && i < 2 * (cy1 - cy0))
      wrow |= 1u << i;
  R tyr[TG];
#pragma unroll
  for (int i = 0; i < TG; ++i)
    tyr[i] = __ldg(&ly[min(cy0 + i, m1 + 1) + 2].t); // odd row 2(cy0+i)+1
  int crow[TG + 1]; // clamped coarse rows
#pragma unroll
  for (int i = 0; i <= TG; ++i)
    crow[i] = min(cy0 + i, m1 - 1);
  int rfo[TG]; // clamped class rank of odd rows
#pragma unroll
  for (int i = 0; i < TG; ++i)
    rfo[i] = min(cy0 + i, max(m1 - 2, 0));

  const int cz0 = Z3 ? int(tzc) * tl.zc : 0;
  const int cz1 = Z3 ? min(cz0 + tl.zc, m2) : 1;
  // step k: even plane 2k (coarse plane k) and, for k > cz0, the odd plane
  // 2k-1 between coarse planes k-1 and k
  const int kend = Z3 ? min(cz1, m2 - 1) : 0;
  // All of a step's inputs -- the TG+1 coarse rows and the 7 TG class rows
  // of both planes -- are loaded in ONE batch at addresses that are always
  // valid (planes clamped; unused values are discarded), so a step exposes
  // one load latency instead of three (ncu: 68 % long-scoreboard stalls on
  // the lerp, shuffle and class-add consumers of three dependent batches);
  // with LEAN_RG_PF the batch of step k+1 is issued before step k computes.
  struct In {
    R c[TG + 1], v[7][TG];
  };
  // 32-bit element indices (lean plans: N < 2^32)
  auto load = [&](int k, In &in) {
    const uint32_t cp = uint32_t(m01) * uint32_t(k) + uint32_t(qe);
#pragma unroll
    for (int i = 0; i <= TG; ++i)
      in.c[i] = __ldg(coarse + (cp + uint32_t(m0 * crow[i])));
    if constexpr (CLS) {
      const uint32_t ke = uint32_t(min(k, m2 - 1)), zr = uint32_t(max(k - 1, 0));
      const uint32_t um0 = uint32_t(m0), um1 = uint32_t(m1);
      const uint32_t c1 = uint32_t(g.tbase[1]) + qo + (um0 - 1) * (um1 * ke);
      const uint32_t c2 = uint32_t(g.tbase[2]) + qe + um0 * ((um1 - 1) * ke);
      const uint32_t c3 = uint32_t(g.tbase[3]) + qo + (um0 - 1) * ((um1 - 1) * ke);
#pragma unroll
      for (int i = 0; i < TG; ++i) {
        in.v[0][i] = __ldg(cls + (c1 + (um0 - 1) * uint32_t(crow[i])));
        in.v[1][i] = __ldg(cls + (c2 + um0 * uint32_t(rfo[i])));
        in.v[2][i] = __ldg(cls + (c3 + (um0 - 1) * uint32_t(rfo[i])));
      }
      if constexpr (Z3) {
        const uint32_t c4 = uint32_t(g.tbase[4]) + qe + um0 * (um1 * zr);
        const uint32_t c5 = uint32_t(g.tbase[5]) + qo + (um0 - 1) * (um1 * zr);
        const uint32_t c6 = uint32_t(g.tbase[6]) + qe + um0 * ((um1 - 1) * zr);
        const uint32_t c7 = uint32_t(g.tbase[7]) + qo + (um0 - 1) * ((um1 - 1) * zr);
#pragma unroll
        for (int i = 0; i < TG; ++i) {
          in.v[3][i] = __ldg(cls + (c4 + um0 * uint32_t(crow[i])));
          in.v[4][i] = __ldg(cls + (c5 + (um0 - 1) * uint32_t(crow[i])));
          in.v[5][i] = __ldg(cls + (c6 + um0 * uint32_t(rfo[i])));
          in.v[6][i] = __ldg(cls + (c7 + (um0 - 1) * uint32_t(rfo[i])));
        }
      }
    }
  };
  R WLe[NF], WLo[NF];
  In cur;
  load(cz0, cur);
  for (int k = cz0; k <= kend; ++k) {
#if LEAN_RG_PF
    In nxt;
    if (k < kend)
      load(k + 1, nxt);
#endif
    R We[NF], Wo[NF];
#pragma unroll
    for (int i = 0; i <= TG; ++i) {
      const R cn = __shfl_down_sync(0xffffffffu, cur.c[i], 1);
      We[2 * i] = cur.c[i];
      Wo[2 * i] = plerp<R, FAST>(cur.c[i], cn, txr);
    }
#pragma unroll
    for (int i = 0; i < TG; ++i) {
      We[2 * i + 1] = plerp<R, FAST>(We[2 * i], We[2 * i + 2], tyr[i]);
      Wo[2 * i + 1] = plerp<R, FAST>(Wo[2 * i], Wo[2 * i + 2], tyr[i]);
    }
    // ---- even plane 2k (written when k < cz1)
    if (k < cz1) {
      const uint32_t op = uint32_t(2 * k) * uint32_t(nxy) + uint32_t(2 * cy0 * n0 + 2 * qc);
#pragma unroll
      for (int i = 0; i < TG; ++i) {
        const R v1 = CLS ? cur.v[0][i] : R(0), v2 = CLS ? cur.v[1][i] : R(0),
                v3 = CLS ? cur.v[2][i] : R(0);
        // even row 2(cy0+i): parity of (2k + 2(cy0+i)) is even -> aligned
        if ((wrow >> (2 * i)) & 1u)
          lean_store_pair<R, true>(out + (op + uint32_t(2 * i * n0)), We[2 * i],
                                   padd<R, FAST>(Wo[2 * i], v1), own, ownO);
        if ((wrow >> (2 * i + 1)) & 1u)
          lean_store_pair<R, false>(out + (op + uint32_t((2 * i + 1) * n0)),
                                    padd<R, FAST>(We[2 * i + 1], v2),
                                    padd<R, FAST>(Wo[2 * i + 1], v3), own, ownO);
      }
    }
    // ---- odd plane 2k-1
    if (Z3 && k > cz0) {
      const R tz = __ldg(&lz[k - 1 + 2].t);
      const uint32_t op =
          uint32_t(2 * k - 1) * uint32_t(nxy) + uint32_t(2 * cy0 * n0 + 2 * qc);
#pragma unroll
      for (int i = 0; i < TG; ++i) {
        const R v4 = CLS ? cur.v[3][i] : R(0), v5 = CLS ? cur.v[4][i] : R(0),
                v6 = CLS ? cur.v[5][i] : R(0), v7 = CLS ? cur.v[6][i] : R(0);
        // odd plane: even rows misaligned, odd rows aligned
        if ((wrow >> (2 * i)) & 1u)
          lean_store_pair<R, false>(
              out + (op + uint32_t(2 * i * n0)),
              padd<R, FAST>(plerp<R, FAST>(WLe[2 * i], We[2 * i], tz), v4),
              padd<R, FAST>(plerp<R, FAST>(WLo[2 * i], Wo[2 * i], tz), v5), own, ownO);
        if ((wrow >> (2 * i + 1)) & 1u)
          lean_store_pair<R, true>(
              out + (op + uint32_t((2 * i + 1) * n0)),
              padd<R, FAST>(plerp<R, FAST>(WLe[2 * i + 1], We[2 * i + 1], tz), v6),
              padd<R, FAST>(plerp<R, FAST>(WLo[2 * i + 1], Wo[2 * i + 1], tz), v7), own,
              ownO);
      }
    }
#pragma unroll
    for (int r = 0; r < NF; ++r) {
      WLe[r] = We[r];
      WLo[r] = Wo[r];
    }
#if LEAN_RG_PF
    cur = nxt;
#else
    if (k < kend)
      load(k + 1, cur);
#endif
  }
}

// z chunk length: the longest (fewest halo planes, kLeanZC) that still
// gives about two full waves of warps; small levels get short chunks so the
// per-warp plane walk (a serial chain of dependent steps) stays short.
#ifndef LEAN_ZC_MIN
#define LEAN_ZC_MIN 1 // measured: 1 beats 2 by 0.3 % of the 1025^3 step (small levels)
#endif
inline int lean_zc(uint64_t xy_tiles, uint32_t m2, bool z3, int zmax = kLeanZC) {
  if (!z3)
    return 1;
#ifndef LEAN_ZC_WANT
#define LEAN_ZC_WANT 32
#endif
  const uint64_t want = 148ull * LEAN_ZC_WANT; // warps
  int zc = zmax;
  while (zc > LEAN_ZC_MIN && xy_tiles * ((m2 + zc - 1) / zc) < want)
    zc /= 2;
  return zc;
}

template <typename R> LeanTiles lean_tiles(uint32_t m0, uint32_t m1, uint32_t m2, bool z3) {
  LeanTiles t;
  t.ntx = (m0 + kLeanOut - 1) / kLeanOut;
  t.nty = (m1 + lean_ty<R>() - 1) / lean_ty<R>();
  t.zc = lean_zc(uint64_t(t.ntx) * t.nty, m2, z3);
  t.ntz = z3 ? (m2 + t.zc - 1) / t.zc : 1;
  return t;
}

template <typename R>
LeanTiles lean_rtiles(uint32_t m0, uint32_t m1, uint32_t m2, bool z3, bool fast = true) {
  LeanTiles t;
  t.ntx = (m0 + kLeanOut - 1) / kLeanOut;
  const int ty = fast ? lean_ty_rl<R, true>() : lean_ty_rl<R, false>();
  t.nty = (m1 + ty - 1) / ty;
  // longer chunks for the load-vector kernel: fewer halo planes re-read
  // (measured 1.205 -> 1.172 ms at 1025^3 f32; the other two are faster at 32)
  t.zc = lean_zc(uint64_t(t.ntx) * t.nty, m2, z3, 2 * kLeanZC);
  t.ntz = z3 ? (m2 + t.zc - 1) / t.zc : 1;
  return t;
}

template <typename R> LeanTiles lean_gtiles(uint32_t m0, uint32_t m1, uint32_t m2, bool z3) {
  LeanTiles t;
  t.ntx = (m0 + kLeanGOut - 1) / kLeanGOut;
  t.nty = (m1 + lean_tg<R>() - 1) / lean_tg<R>();
  t.zc = lean_zc(uint64_t(t.ntx) * t.nty, m2, z3);
  t.ntz = z3 ? (m2 + t.zc - 1) / t.zc : 1;
  return t;
}

} // namespace mgrg
