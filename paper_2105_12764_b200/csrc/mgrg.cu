// mgrg.cu -- plan, level loop and C ABI (include/mgrg.h) of the B200 path.
//
// Host side of the drop-in boundary: the reference engine
// (RefactorEngine<Real>, /root/reference/proj/include/mgr/refactor.hpp:153-458)
// becomes a plan (hierarchy + geometry + workspace on the device) and a level
// loop that launches, per level,
//   decompose: dec_level -> thomas(d) for every refining d (last one fused
//              with apply_pack, writing the packed level-(l-1) array);
//   recompose: rec_load -> thomas(d) (last fused with unapply_expand) ->
//              rec_gpk (scatter_class + GPK inverse, writing the level-l
//              array).
// Level arrays live in HBM packed row-major (paper §III.C "stride always
// one"); the class buffer is the single N-element output.
#include <algorithm>
#include <array>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/mgrg.h"
#include "kernels.cuh"
#include "kernels2.cuh"
#include "thomas.cuh"
#include "thomas_scan.cuh"
#include "kernels3.cuh"
#include "kernels4.cuh"
#include "lean.cuh"
#include "thomas_fiber.cuh"
#include "thomas_exact.cuh"
#include "thomas_2pass.cuh"
#include "gen4.cuh"
#include "hostio.cuh"

using namespace mgrg;

namespace {

thread_local std::string g_last_error;

mgrg_status fail(mgrg_status st, const std::string &msg) {
  g_last_error = msg;
  return st;
}

#define CUDA_TRY(expr)                                                         \
  do {                                                                         \
    cudaError_t e_ = (expr);                                                   \
    if (e_ != cudaSuccess)                                                     \
      return fail(MGRG_CUDA_ERROR, std::string(#expr) + ": " +                 \
                                       cudaGetErrorString(e_));                \
  } while (0)

constexpr int kMaxLevels = 40;

// RAII current-device switch: the C ABI may be called from threads whose
// current device differs from the plan's.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev)
      cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev)
      cudaSetDevice(prev);
  }
};

uint64_t coarse_extent(uint64_t n) { return n / 2 + 1; } // grid.hpp:77

// Host hierarchy: build_hierarchy / build_dim_levels (grid.cpp:40-112) with
// the validation of validate_grid_geometry (grid.cpp:14-36).
struct Hierarchy {
  int nd = 0;
  int L = 0;
  uint64_t shape[4] = {1, 1, 1, 1};
  std::vector<std::vector<uint64_t>> ext;             // [l][d]
  std::vector<std::vector<std::vector<double>>> h, r; // [d][l][i]
  std::vector<std::vector<double>> coords;            // [d][i], finest level (MGRF header)
};

mgrg_status build_hierarchy(const mgrg_grid_desc &desc, Hierarchy &H) {
  const int nd = desc.ndims;
  if (nd < 1 || nd > 4)
    return fail(MGRG_INVALID_GRID, "grid must have 1..4 dimensions, got " +
                                       std::to_string(nd));
  H.nd = nd;
  std::vector<std::vector<double>> coords(nd);
  const double *cp = desc.coords;
  for (int d = 0; d < nd; ++d) {
    const uint64_t n = desc.shape[d];
    H.shape[d] = n;
    if (n < 2)
      return fail(MGRG_INVALID_GRID, "dimension " + std::to_string(d) + " has " +
                                         std::to_string(n) +
                                         " nodes; need at least 2");
    if (n > (uint64_t(1) << 31))
      return fail(MGRG_UNSUPPORTED, "extent too large");
    coords[d].resize(n);
    for (uint64_t i = 0; i < n; ++i)
      coords[d][i] = cp ? cp[i] : (n > 1 ? double(i) / double(n - 1) : 0.0);
    if (cp)
      cp += n;
    for (uint64_t i = 0; i + 1 < n; ++i)
      if (!(coords[d][i] < coords[d][i + 1]))
        return fail(MGRG_INVALID_GRID, "coordinates of dimension " +
                                           std::to_string(d) +
                                           " are not strictly increasing at index " +
                                           std::to_string(i));
  }
  H.coords = coords;
  int levels = 0;
  bool any = false;
  for (int d = 0; d < nd; ++d) {
    const uint64_t e = desc.shape[d];
    if (e < 3)
      continue;
    const int depth = int(std::floor(std::log2(double(e - 1))));
    levels = any ? std::min(levels, depth) : depth;
    any = true;
  }
  if (!any)
    return fail(MGRG_INVALID_GRID, "no dimension has at least 3 nodes");
  if (desc.levels < 0)
    return fail(MGRG_INVALID_LEVEL, "level count must be at least 1");
  if (desc.levels > 0)
    levels = std::min(levels, int(desc.levels));
  if (levels > kMaxLevels)
    return fail(MGRG_UNSUPPORTED, "too many levels");
  H.L = levels;
  H.ext.assign(levels + 1, std::vector<uint64_t>(nd));
  H.h.assign(nd, {});
  H.r.assign(nd, {});
  for (int d = 0; d < nd; ++d) {
    std::vector<std::vector<uint64_t>> idx(levels + 1);
    idx[levels].resize(desc.shape[d]);
    for (uint64_t i = 0; i < desc.shape[d]; ++i)
      idx[levels][i] = i;
    for (int l = levels - 1; l >= 0; --l) {
      const auto &fine = idx[l + 1];
      auto &c = idx[l];
      for (size_t p = 0; p < fine.size(); p += 2)
        c.push_back(fine[p]);
      if (c.back() != fine.back())
        c.push_back(fine.back());
    }
    H.h[d].resize(levels + 1);
    H.r[d].resize(levels + 1);
    for (int l = 0; l <= levels; ++l) {
      const auto &ids = idx[l];
      H.ext[l][d] = ids.size();
      auto &h = H.h[d][l];
      auto &r = H.r[d][l];
      h.resize(ids.size() - 1);
      for (size_t i = 0; i + 1 < ids.size(); ++i)
        h[i] = coords[d][ids[i + 1]] - coords[d][ids[i]];
      if (h.size() >= 2) {
        r.resize(h.size() - 1);
        for (size_t i = 0; i + 1 < h.size(); ++i)
          r[i] = h[i] / (h[i] + h[i + 1]);
      }
    }
  }
  return MGRG_OK;
}

// Tile shapes of the level kernels (coarse outputs per CTA along x, y).
enum class TileKind { t32x8, t128x1 };

struct LaunchCount {
  uint64_t n = 0;
};

template <typename R> struct PlanT {
  std::vector<LevelGeom<R>> geom;                 // [l], l = 1..L
  std::vector<std::array<ThomasGeom<R>, 3>> thom; // [l][kd] (level-(l-1) factors)
  std::vector<std::array<const Stencil<R> *, 3>> sten; // [l][kd] merged R*M tables
  std::vector<std::array<const LeanW<R> *, 3>> lean;   // [l][kd] lean tables (padded)
  std::vector<std::array<ThomasLean<R>, 3>> tlean;     // [l][kd] chunked Thomas tables
  std::vector<std::array<ThomasTP<R>, 3>> ttp;         // [l][kd] two-pass long-fiber tables
  std::vector<Gen4Geom<R>> g4;                         // [l] 4-D levels (gen4.cuh)
  R *d_geom = nullptr;
};

} // namespace

struct mgrg_plan {
  int device = 0;
  int dtype = MGRG_F32;
  int esize = 4;
  Hierarchy H;
  int kmap[3] = {0, -1, -1};              // kernel dim -> user dim (-1 = pad)
  std::vector<std::array<uint32_t, 3>> kext; // [l][kd] padded extents
  std::vector<uint64_t> nodes;            // N_l
  uint32_t refine = 0;                    // kernel-dim refine mask (same at every level)
  int refine_dims[3];
  int nrefine = 0;
  TileKind tile = TileKind::t32x8;
  bool pair_path = false; // x and y refine: pair-lane kernels (kernels2.cuh)
  bool fast = false;      // MGRG_FLAG_FAST: FMA arithmetic policy
  uint32_t zchunk = 32;
  bool lean = false;      // dyadic x/y(/z) refinement: lean warp-tiled kernels (lean.cuh)
  bool gen = false;       // 4-D grid: generic per-pass kernels (gen4.cuh)
  uint64_t offW = 0, offW2 = 0; // gen: two level-L lattices (vec(C) field, mass ping-pong)
  mgrg_status deferred = MGRG_OK;         // SingularSystem found at build time
  std::string deferred_msg;
  PlanT<float> pf;
  PlanT<double> pd;
  void *d_geom = nullptr;
  size_t geom_bytes = 0;
  void *d_ws = nullptr; // [A: N_{L-1}][B: N_{L-2}][F: N_{L-1}]
  size_t ws_bytes = 0;
  uint64_t offA = 0, offB = 0, offF = 0; // element offsets inside d_ws
  uint64_t offTP = 0;                    // two-pass Thomas scratch (thomas_2pass.cuh)
  void *d_stage = nullptr;               // host-API staging (2N elements), lazy
  cudaStream_t own_stream = nullptr;
  cudaStream_t s_in = nullptr, s_out = nullptr; // host-API copy streams (pipelined path)
  cudaEvent_t ev_in[16] = {}, ev_dec[16] = {}, ev_done = nullptr;
  std::unique_ptr<mgrg::HostXfer> xfer; // pinned rings for pageable host buffers
  uint64_t last_launches = 0;
  // per-launch profiling (mgrg_plan_set_profiling)
  bool profiling = false;
  int prof_min_level = 0; // profile launches of levels >= this one only
  struct Prof {
    int kind, level;
    uint64_t bytes;
    cudaEvent_t e0, e1;
  };
  std::vector<Prof> prof;
  std::vector<cudaEvent_t> event_pool;
  size_t prof_used = 0;
  // CUDA-graph replay of the level loop (mgrg_plan_set_graphs): one
  // instantiated graph per (operation, buffers, k), most recent last
  int split_op = 0; // host begin/end pair in flight: 1 decompose, 2 recompose
  bool graphs = false;
  struct Graph {
    int op; // 0 decompose, 1 recompose
    const void *a;
    void *b;
    int32_t k;
    cudaGraphExec_t exec;
    uint64_t launches;
  };
  std::vector<Graph> graph_cache;
  cudaStream_t graph_stream = nullptr;
  cudaEvent_t graph_ev[2] = {nullptr, nullptr};
};

namespace {

template <typename R> PlanT<R> &pt(mgrg_plan *p);
template <> PlanT<float> &pt<float>(mgrg_plan *p) { return p->pf; }
template <> PlanT<double> &pt<double>(mgrg_plan *p) { return p->pd; }

// make_class_layout (grid.cpp:140-165) on the padded 3-D lattice.
template <typename R>
void fill_layout(LevelGeom<R> &g) {
  uint64_t off = 0;
  g.tbase[0] = 0;
  g.tex[0] = g.tey[0] = 0;
  for (unsigned mask = 1; mask < 8; ++mask) {
    uint64_t e[3], count = 1;
    for (int d = 0; d < 3; ++d) {
      const uint64_t n = g.n[d];
      e[d] = ((mask >> d) & 1) ? n - coarse_extent(n) : coarse_extent(n);
      count *= e[d];
    }
    g.tbase[mask] = off;
    g.tex[mask] = uint32_t(e[0]);
    g.tey[mask] = uint32_t(e[1]);
    off += count;
  }
}

// TridiagonalOperator::build (kernels.hpp:107-135) in the working precision.
template <typename R>
bool thomas_factors(const std::vector<double> &hd, std::vector<R> &h,
                    std::vector<R> &fwd, std::vector<R> &ip, std::string &err) {
  const size_t n = hd.size() + 1;
  h.resize(hd.size());
  for (size_t i = 0; i < hd.size(); ++i)
    h[i] = R(hd[i]);
  fwd.assign(n, R(0));
  ip.assign(n, R(0));
  R pivot = R(2) * h[0];
  if (!(pivot > R(0))) {
    err = "nonpositive leading pivot";
    return false;
  }
  ip[0] = R(1) / pivot;
  for (size_t i = 1; i < n; ++i) {
    const R sub = h[i - 1];
    fwd[i] = -sub * ip[i - 1];
    const R diag = i + 1 < n ? R(2) * (h[i - 1] + h[i]) : R(2) * h[i - 1];
    pivot = diag + fwd[i] * sub;
    if (!(pivot > R(0))) {
      err = "nonpositive pivot at row " + std::to_string(i);
      return false;
    }
    ip[i] = R(1) / pivot;
  }
  return true;
}

// Merged mass-trans coefficients of coarse output c along one dimension of
// extent n (masstrans_window, kernels.hpp:159-178), computed in the working
// precision exactly as the reference forms them: h cast to R, then
// 2*(h[j-1]+h[j]), 2*h[0], 1 - r[q] in R.
template <typename R>
Stencil<R> make_stencil(const std::vector<double> &hd, const std::vector<double> &rd,
                        uint64_t n, uint64_t c, bool allow_shift) {
  auto h = [&](uint64_t i) { return R(hd[i]); };
  auto r = [&](uint64_t i) { return R(rd[i]); };
  auto dd = [&](uint64_t j) { return R(R(2) * R(h(j - 1) + h(j))); };
  auto coarse = [&](uint64_t p) { return p % 2 == 0 || p == n - 1; };
  const uint64_t q = std::min<uint64_t>(2 * c, n - 1);
  Stencil<R> s{};
  uint32_t fl = ST_VALID;
  if (q == 0) {
    fl |= ST_LEFT;
    s.d0 = R(R(2) * h(0));
    s.h0 = h(0);
  } else if (q == n - 1) {
    fl |= ST_RIGHT;
    s.hm1 = h(n - 2);
    s.d0 = R(R(2) * h(n - 2));
  } else {
    s.hm1 = h(q - 1);
    s.d0 = dd(q);
    s.h0 = h(q);
  }
  if (q >= 1 && !coarse(q - 1)) {
    fl |= ST_HASL;
    s.hm2 = h(q - 2);
    s.dm1 = dd(q - 1);
    s.hm1 = h(q - 1);
    s.cl = r(q - 2);
  }
  if (q + 1 < n && !coarse(q + 1)) {
    fl |= ST_HASR;
    s.h0 = h(q);
    s.dp1 = dd(q + 1);
    s.hp1 = h(q + 1);
    s.cr = R(R(1) - r(q));
  }
  // fast path: the merged 5-tap weights, formed in fp64 from the fp64
  // geometry and rounded once
  double wq[5] = {0, 0, 0, 0, 0}; // positions q-2 .. q+2
  auto H = [&](uint64_t i) { return hd[i]; };
  if (q == 0) {
    wq[2] += 2 * H(0);
    wq[3] += H(0);
  } else if (q == n - 1) {
    wq[1] += H(n - 2);
    wq[2] += 2 * H(n - 2);
  } else {
    wq[1] += H(q - 1);
    wq[2] += 2 * (H(q - 1) + H(q));
    wq[3] += H(q);
  }
  if (fl & ST_HASL) {
    const double cl = rd[q - 2];
    wq[0] += cl * H(q - 2);
    wq[1] += cl * 2 * (H(q - 2) + H(q - 1));
    wq[2] += cl * H(q - 1);
  }
  if (fl & ST_HASR) {
    const double cr = 1.0 - rd[q];
    wq[2] += cr * H(q);
    wq[3] += cr * 2 * (H(q) + H(q + 1));
    wq[4] += cr * H(q + 1);
  }
  const bool shift = allow_shift && q != 2 * c;
  for (int t = 0; t < 5; ++t) {
    // taps are relative to the nominal centre 2c (x, y) or q (z); wq[s] sits
    // at q-2+s, so with q = 2c-1 (shift) tap t takes wq[t+1]
    const int src = shift ? t + 1 : t; // tap t sits at 2c-2+t = q-1+t
    s.w[t] = (src >= 0 && src < 5) ? R(wq[src]) : R(0);
  }
  if (shift)
    fl |= ST_SHIFT;
  s.flags = fl;
  return s;
}

int knob(const char *name, int dflt);
// two-pass long-fiber Thomas (thomas_2pass.cuh) for FAST strided (y / z)
// fibers of at least this many positions; the cluster kernel serves x fibers
// and shorter ones.  Measured (profiles/r2/tuning/README.md, 8193^2 f64):
// y at m = 4097 150 -> 112 us; at m = 2049 35 -> 40 us and x fibers at m =
// 4097 124 -> 135 us (the DIM-0 passes transpose through shared memory).
int g_tp_min = knob("MGRG_TP_MIN", 4097);

template <typename R> mgrg_status upload_geometry(mgrg_plan *p) {
  const Hierarchy &H = p->H;
  const int L = H.L;
  // host staging of every per-level array in R, then one upload
  std::vector<R> buf;
  struct Ref {
    size_t h[3], r[3], th[3], tf[3], ti[3], st[3], lw[3], tl[3], tp[3];
  };
  std::vector<Ref> refs(L + 1);
  auto push = [&](const std::vector<R> &v) {
    size_t off = buf.size();
    buf.insert(buf.end(), v.begin(), v.end());
    buf.resize((buf.size() + 31) & ~size_t(31), R(0)); // 256-byte alignment
    return off;
  };
  std::vector<std::array<ThomasGeom<R>, 3>> thom(L + 1);
  for (int l = 1; l <= L; ++l) {
    for (int kd = 0; kd < 3; ++kd) {
      refs[l].h[kd] = refs[l].r[kd] = refs[l].th[kd] = refs[l].tf[kd] =
          refs[l].ti[kd] = refs[l].st[kd] = refs[l].lw[kd] = refs[l].tl[kd] = refs[l].tp[kd] = size_t(-1);
      const int ud = p->kmap[kd];
      if (ud < 0)
        continue;
      std::vector<R> h(H.h[ud][l].begin(), H.h[ud][l].end());
      std::vector<R> r(H.r[ud][l].begin(), H.r[ud][l].end());
      refs[l].h[kd] = push(h);
      refs[l].r[kd] = push(r);
      if (H.ext[l - 1][ud] < H.ext[l][ud]) {
        std::vector<R> th, tf, ti;
        std::string err;
        if (!thomas_factors<R>(H.h[ud][l - 1], th, tf, ti, err) &&
            p->deferred == MGRG_OK) {
          p->deferred = MGRG_SINGULAR_SYSTEM;
          p->deferred_msg = err;
        }
        if (th.empty())
          th.push_back(R(0));
        refs[l].th[kd] = push(th);
        refs[l].tf[kd] = push(tf);
        refs[l].ti[kd] = push(ti);
        {
          // chunked-Thomas tables (thomas_fiber.cuh): {fwd, ip, g, PF, PB}
          // per position (8-padded), PFend, PBstart [tf_nch]; products in
          // fp64 from the working-precision factors, rounded once
          const uint32_t mm = uint32_t(tf.size());
          std::vector<R> tl(tf_tab_elems<R>(mm, kd), R(0));
          const int nch = std::max(tf_nch<R>(mm, kd), 1), ch = std::max(tf_ch<R>(mm, kd), 1);
          const uint32_t mp = std::max<uint32_t>(uint32_t(nch) * uint32_t(ch), mm);
          R *Q = tl.data(), *Tpe = Q + 8 * size_t(mp), *Tps = Tpe + nch;
          for (uint32_t i = 0; i < mp; ++i) { // padding: fwd = g = 0, ip = 1
            const bool real = i < mm;
            Q[8 * i] = real ? tf[i] : R(0);
            Q[8 * i + 1] = real ? ti[i] : R(1);
            Q[8 * i + 2] = (i + 1 < mm) ? R(-double(ti[i]) * double(th[i])) : R(0);
          }
          for (int w = 0; w < tf_nch<R>(mm, kd); ++w) {
            const uint32_t a = uint32_t(w) * uint32_t(ch), b = a + uint32_t(ch);
            double pr = 1.0;
            for (uint32_t i = a; i < b; ++i) {
              pr *= double(Q[8 * i]);
              Q[8 * i + 3] = R(pr);
            }
            Tpe[w] = R(pr);
            pr = 1.0;
            for (uint32_t i = b; i > a; --i) {
              pr *= double(Q[8 * (i - 1) + 2]);
              Q[8 * (i - 1) + 4] = R(pr);
            }
            Tps[w] = R(pr);
          }
          // cluster-segment multipliers (thomas_cluster_kernel): products of
          // the per-position factors over each CTA's segment
          if (tf_cl<R>(mm, kd) > 1) {
            const int cl = tf_cl<R>(mm, kd);
            const uint32_t seg = uint32_t(tf_nw<R>(mm, kd)) * uint32_t(ch);
            R *Tmf = Tps + nch, *Tmb = Tmf + cl;
            for (int r = 0; r < cl; ++r) {
              double pf = 1.0, pb = 1.0;
              for (uint32_t i = uint32_t(r) * seg; i < uint32_t(r + 1) * seg; ++i) {
                pf *= double(Q[8 * i]);
                pb *= double(Q[8 * i + 2]);
              }
              Tmf[r] = R(pf);
              Tmb[r] = R(pb);
            }
          }
          refs[l].tl[kd] = push(tl);
        }
        if (kd != 0 && tf.size() >= size_t(g_tp_min) && tf.size() <= size_t(kTpC) * kTpMaxK) {
          // two-pass long-fiber tables (thomas_2pass.cuh): {fwd, ip, g, 0} per
          // position, {PF, Q, PB, 0} per 32-position chunk; products in fp64
          // from the working-precision factors, rounded once
          const uint32_t mm = uint32_t(tf.size()), K = (mm + kTpC - 1) / kTpC;
          std::vector<R> tq(4 * size_t(mm) + 4 * size_t(K), R(0));
          R *Q = tq.data(), *Ck = Q + 4 * size_t(mm);
          for (uint32_t i = 0; i < mm; ++i) {
            Q[4 * i] = tf[i];
            Q[4 * i + 1] = ti[i];
            Q[4 * i + 2] = (i + 1 < mm) ? R(-double(ti[i]) * double(th[i])) : R(0);
          }
          for (uint32_t k = 0; k < K; ++k) {
            const uint32_t a = k * kTpC, b = std::min(mm, a + kTpC);
            double pf = 1.0, pb = 1.0, x = 0.0;
            std::vector<double> pfi(b - a);
            for (uint32_t i = a; i < b; ++i) {
              pf *= double(Q[4 * i]);
              pfi[i - a] = pf;
            }
            for (uint32_t i = b; i > a; --i) {
              const uint32_t j = i - 1;
              x = double(Q[4 * j + 1]) * pfi[j - a] + (j + 1 < b ? double(Q[4 * j + 2]) * x : 0.0);
              pb *= double(Q[4 * j + 2]);
            }
            Ck[4 * k] = R(pf);
            Ck[4 * k + 1] = R(x);
            Ck[4 * k + 2] = R(pb);
          }
          refs[l].tp[kd] = push(tq);
        }
        // stencil table (raw bytes of Stencil<R>, a whole number of R's)
        const uint64_t n = H.ext[l][ud], m = H.ext[l - 1][ud];
        std::vector<R> raw(m * (sizeof(Stencil<R>) / sizeof(R)));
        for (uint64_t c = 0; c < m; ++c) {
          const Stencil<R> st = make_stencil<R>(H.h[ud][l], H.r[ud][l], n, c, kd < 2);
          std::memcpy(raw.data() + c * (sizeof(Stencil<R>) / sizeof(R)), &st, sizeof(st));
        }
        refs[l].st[kd] = push(raw);
        // lean table: entry c+2 for c in [-2, m+1]; FAST weights + odd-node ratio
        constexpr size_t LW = sizeof(LeanW<R>) / sizeof(R);
        std::vector<R> lw((m + 4) * LW, R(0));
        for (uint64_t c = 0; c < m; ++c) {
          const Stencil<R> st = make_stencil<R>(H.h[ud][l], H.r[ud][l], n, c, kd < 2);
          LeanW<R> e{};
          for (int t = 0; t < 5; ++t)
            e.w[t] = st.w[t];
          e.t = 2 * c + 1 < n - 1 ? R(H.r[ud][l][2 * c]) : R(0);
          std::memcpy(lw.data() + (c + 2) * LW, &e, sizeof(e));
        }
        refs[l].lw[kd] = push(lw);
      }
    }
  }
  if (buf.empty())
    buf.resize(32, R(0));
  p->geom_bytes = buf.size() * sizeof(R);
  CUDA_TRY(cudaMalloc(&p->d_geom, p->geom_bytes));
  CUDA_TRY(cudaMemcpy(p->d_geom, buf.data(), p->geom_bytes, cudaMemcpyHostToDevice));
  R *base = static_cast<R *>(p->d_geom);
  PlanT<R> &P = pt<R>(p);
  P.geom.assign(L + 1, LevelGeom<R>{});
  P.thom.assign(L + 1, {});
  P.sten.assign(L + 1, {nullptr, nullptr, nullptr});
  P.lean.assign(L + 1, {nullptr, nullptr, nullptr});
  P.tlean.assign(L + 1, {});
  P.ttp.assign(L + 1, {});
  for (int l = 1; l <= L; ++l) {
    LevelGeom<R> &g = P.geom[l];
    g.refine = 0;
    for (int kd = 0; kd < 3; ++kd) {
      g.n[kd] = p->kext[l][kd];
      g.m[kd] = p->kext[l - 1][kd];
      if (g.m[kd] < g.n[kd])
        g.refine |= 1u << kd;
      g.h[kd] = refs[l].h[kd] == size_t(-1) ? nullptr : base + refs[l].h[kd];
      g.r[kd] = refs[l].r[kd] == size_t(-1) ? nullptr : base + refs[l].r[kd];
      ThomasGeom<R> &t = P.thom[l][kd];
      t.m = g.m[kd];
      t.h = refs[l].th[kd] == size_t(-1) ? nullptr : base + refs[l].th[kd];
      t.fwd = refs[l].tf[kd] == size_t(-1) ? nullptr : base + refs[l].tf[kd];
      t.ip = refs[l].ti[kd] == size_t(-1) ? nullptr : base + refs[l].ti[kd];
      P.sten[l][kd] = refs[l].st[kd] == size_t(-1)
                          ? nullptr
                          : reinterpret_cast<const Stencil<R> *>(base + refs[l].st[kd]);
      if (refs[l].tl[kd] != size_t(-1)) {
        ThomasLean<R> &q = P.tlean[l][kd];
        const uint32_t mm = g.m[kd];
        const R *b0 = base + refs[l].tl[kd];
        q.m = mm;
        q.tab = b0;
      }
      if (refs[l].tp[kd] != size_t(-1)) {
        ThomasTP<R> &q = P.ttp[l][kd];
        q.m = g.m[kd];
        q.K = (q.m + kTpC - 1) / kTpC;
        q.q = base + refs[l].tp[kd];
        q.ck = q.q + 4 * size_t(q.m);
      }
      P.lean[l][kd] = refs[l].lw[kd] == size_t(-1)
                          ? nullptr
                          : reinterpret_cast<const LeanW<R> *>(base + refs[l].lw[kd]);
    }
    fill_layout(g);
  }
  return MGRG_OK;
}

// 4-D plans (gen4.cuh): per level the spacings/ratios of every dimension,
// the level-(l-1) Thomas factors of the refining ones and the class layout
// (make_class_layout, grid.cpp:140-165) over all four dimensions.
template <typename R> mgrg_status upload_geometry_gen(mgrg_plan *p) {
  const Hierarchy &H = p->H;
  const int L = H.L;
  std::vector<R> buf;
  auto push = [&](const std::vector<R> &v) {
    size_t off = buf.size();
    buf.insert(buf.end(), v.begin(), v.end());
    buf.resize((buf.size() + 31) & ~size_t(31), R(0));
    return off;
  };
  constexpr size_t kNone = size_t(-1);
  struct Ref {
    size_t h[kGenDims], r[kGenDims], th[kGenDims], tf[kGenDims], ti[kGenDims];
  };
  std::vector<Ref> refs(L + 1);
  for (int l = 1; l <= L; ++l)
    for (int d = 0; d < kGenDims; ++d) {
      Ref &f = refs[l];
      f.h[d] = f.r[d] = f.th[d] = f.tf[d] = f.ti[d] = kNone;
      std::vector<R> h(H.h[d][l].begin(), H.h[d][l].end());
      std::vector<R> r(H.r[d][l].begin(), H.r[d][l].end());
      f.h[d] = push(h);
      f.r[d] = push(r);
      if (H.ext[l - 1][d] < H.ext[l][d]) {
        std::vector<R> th, tf, ti;
        std::string err;
        if (!thomas_factors<R>(H.h[d][l - 1], th, tf, ti, err) && p->deferred == MGRG_OK) {
          p->deferred = MGRG_SINGULAR_SYSTEM;
          p->deferred_msg = err;
        }
        if (th.empty())
          th.push_back(R(0));
        f.th[d] = push(th);
        f.tf[d] = push(tf);
        f.ti[d] = push(ti);
      }
    }
  if (buf.empty())
    buf.resize(32, R(0));
  p->geom_bytes = buf.size() * sizeof(R);
  CUDA_TRY(cudaMalloc(&p->d_geom, p->geom_bytes));
  CUDA_TRY(cudaMemcpy(p->d_geom, buf.data(), p->geom_bytes, cudaMemcpyHostToDevice));
  const R *base = static_cast<const R *>(p->d_geom);
  auto at = [&](size_t o) { return o == kNone ? nullptr : base + o; };
  PlanT<R> &P = pt<R>(p);
  P.g4.assign(L + 1, Gen4Geom<R>{});
  for (int l = 1; l <= L; ++l) {
    Gen4Geom<R> &g = P.g4[l];
    for (int d = 0; d < kGenDims; ++d) {
      g.n[d] = uint32_t(H.ext[l][d]);
      g.m[d] = uint32_t(H.ext[l - 1][d]);
      g.fn[d] = make_fastdiv(g.n[d]);
      g.fm[d] = make_fastdiv(g.m[d]);
      g.h[d] = at(refs[l].h[d]);
      g.r[d] = at(refs[l].r[d]);
      g.th[d] = at(refs[l].th[d]);
      g.tf[d] = at(refs[l].tf[d]);
      g.ti[d] = at(refs[l].ti[d]);
    }
    uint64_t off = 0;
    g.tbase[0] = 0;
    for (unsigned mask = 1; mask < (1u << kGenDims); ++mask) {
      uint64_t count = 1;
      for (int d = 0; d < kGenDims; ++d) {
        const uint64_t n = g.n[d];
        g.cext[mask][d] = uint32_t(((mask >> d) & 1) ? n - coarse_extent(n) : coarse_extent(n));
        count *= g.cext[mask][d];
      }
      g.tbase[mask] = off;
      off += count;
    }
  }
  return MGRG_OK;
}

template <typename R, int CX, int CY> void set_smem_attrs() {
  static bool done = false; // per instantiation; attribute is per device too
  (void)done;
  cudaFuncSetAttribute(dec_level_kernel<R, CX, CY>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(dec_level_smem<R, CX, CY>()));
  cudaFuncSetAttribute(rec_load_kernel<R, CX, CY>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(rec_load_smem<R, CX, CY>()));
  cudaFuncSetAttribute(rec_gpk_kernel<R, CX, CY>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(rec_gpk_smem<R, CX, CY>()));
}

template <typename R, int CX, int CY>
dim3 level_grid(const LevelGeom<R> &g, uint32_t zchunk) {
  return dim3((g.m[0] + CX - 1) / CX, (g.m[1] + CY - 1) / CY,
              (g.m[2] + zchunk - 1) / zchunk);
}

template <typename R, int CX, int CY>
void launch_dec_level(const LevelGeom<R> &g, const R *in, R *cls, R *P, R *f,
                      uint32_t zchunk, cudaStream_t s) {
  dec_level_kernel<R, CX, CY><<<level_grid<R, CX, CY>(g, zchunk), CX * CY,
                                dec_level_smem<R, CX, CY>(), s>>>(g, in, cls, P, f,
                                                                  zchunk);
}
template <typename R, int CX, int CY>
void launch_rec_load(const LevelGeom<R> &g, const R *cls, R *f, uint32_t zchunk,
                     cudaStream_t s) {
  rec_load_kernel<R, CX, CY><<<level_grid<R, CX, CY>(g, zchunk), CX * CY,
                               rec_load_smem<R, CX, CY>(), s>>>(g, cls, f, zchunk);
}
template <typename R, int CX, int CY>
void launch_rec_gpk(const LevelGeom<R> &g, const R *coarse, const R *cls, R *out,
                    uint32_t zchunk, cudaStream_t s) {
  rec_gpk_kernel<R, CX, CY><<<level_grid<R, CX, CY>(g, zchunk), CX * CY,
                              rec_gpk_smem<R, CX, CY>(), s>>>(g, coarse, cls, out,
                                                              zchunk);
}

static_assert(sizeof(Stencil<float>) % sizeof(float) == 0, "stencil layout");
static_assert(sizeof(Stencil<double>) % sizeof(double) == 0, "stencil layout");

// Tuning / A-B knobs.  Release builds use the measured defaults and never
// read the environment; a debug build (-DMGRG_DEBUG_KNOBS) lets an A/B run
// override a knob.  No knob changes a value-affecting contract (the
// arithmetic policy is the caller's MGRG_FLAG_FAST, nothing else).
int knob(const char *name, int dflt) {
#ifdef MGRG_DEBUG_KNOBS
  if (const char *e = std::getenv(name))
    return std::atoi(e);
#endif
  (void)name;
  return dflt;
}
// chunked fiber-resident Thomas (MGRG_TFIBER=0 disables)
int g_thomas_fiber = knob("MGRG_TFIBER", 1);
// Profiling event record: inside a stream capture (graph replay mode) the
// record must be an EXTERNAL event-record node to be timeable.
cudaError_t prof_record(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  return cs == cudaStreamCaptureStatusActive
             ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
             : cudaEventRecord(e, s);
}
// programmatic dependent launch of the level-loop kernels (MGRG_PDL=0 disables)
int g_pdl = knob("MGRG_PDL", 1);

// Launch with programmatic stream serialization: the kernel's CTAs may be
// scheduled before its stream predecessor has finished; the kernel waits in
// pdl_wait() (common.cuh) before touching any data.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// exact-policy resident Thomas (thomas_exact.cuh; MGRG_TEXACT=0 disables,
// 2 also uses it for y / z fibers)
int g_thomas_exact = knob("MGRG_TEXACT", 1);
// pipelined host-buffer decompose (MGRG_PIPELINE=0 disables)
int g_pipelined_host = knob("MGRG_PIPELINE", 1);
// experiment knob: one-launch Thomas for small lattices (MGRG_TSMALL=0 disables)
int g_thomas_small = knob("MGRG_TSMALL", 1);
constexpr uint32_t kZChunk = 32; // coarse-z planes per CTA of the pair-lane kernels
template <typename R> constexpr int pair_cy() { return sizeof(R) == 4 ? 16 : 8; }

template <typename R, int CY, bool FAST> void set_pair_attrs_t() {
  cudaFuncSetAttribute(rl2_kernel<R, CY, FAST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(rl2_smem<R, CY>()));
  cudaFuncSetAttribute(rg2_kernel<R, CY, FAST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(rg2_smem<R, CY>()));
}
template <typename R, int CY> void set_pair_attrs() {
  set_pair_attrs_t<R, CY, false>();
  set_pair_attrs_t<R, CY, true>();
  // the lean decompose ring (f64 bands above 2 coarse rows exceed 48 KB)
  for (auto k : {lean_dec_kernel<R, true, true>, lean_dec_kernel<R, true, false>,
                 lean_dec_kernel<R, false, true>, lean_dec_kernel<R, false, false>})
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(lean_dec_smem<R>()));
  cudaFuncSetAttribute(dec4_kernel<R, cy4<R>(), false>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(dec4_smem<R, cy4<R>()>()));
  cudaFuncSetAttribute(dec4_kernel<R, cy4<R>(), true>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(dec4_smem<R, cy4<R>()>()));
}

template <typename R> dim3 pair_grid(const LevelGeom<R> &g, uint32_t cx) {
  constexpr int CY = pair_cy<R>();
  const uint32_t ntz = (g.refine & 4) ? (g.m[2] + kZChunk - 1) / kZChunk : g.m[2];
  return dim3((g.m[0] + cx - 1) / cx, (g.m[1] + CY - 1) / CY, ntz);
}

template <typename R>
void launch_dec4(bool fast, const LevelGeom<R> &g,
                 const std::array<const Stencil<R> *, 3> &st, const R *in, R *cls, R *P,
                 R *f, cudaStream_t s) {
  constexpr int CY = cy4<R>();
  const uint32_t ntz = (g.refine & 4) ? (g.m[2] + kZChunk - 1) / kZChunk : g.m[2];
  const dim3 grid((g.m[0] + 29) / 30, (g.m[1] + CY - 1) / CY, ntz);
  auto k = fast ? dec4_kernel<R, CY, true> : dec4_kernel<R, CY, false>;
  k<<<grid, 256, dec4_smem<R, CY>(), s>>>(g, st[0], st[1], st[2], in, cls, P, f, grid.x,
                                          grid.y, grid.z);
}
template <typename R> bool lean_out_ok(const R *out) {
  return (reinterpret_cast<uintptr_t>(out) & (2 * sizeof(R) - 1)) == 0;
}
template <typename R> bool lean_level(const LevelGeom<R> &g) {
  return (g.n[0] & 1u) && (g.n[1] & 1u) && (g.n[2] & 1u);
}
template <typename R>
void launch_lean_dec(bool fast, const LevelGeom<R> &g, const std::array<const LeanW<R> *, 3> &st,
                     const std::array<const Stencil<R> *, 3> &sc, const R *in, R *cls, R *P,
                     R *f, cudaStream_t s) {
  const bool z3 = g.n[2] > 1;
  const LeanTiles t = lean_tiles<R>(g.m[0], g.m[1], g.m[2], z3);
  const unsigned blocks = unsigned((t.warps() + kLeanWPB - 1) / kLeanWPB);
  auto k = z3 ? (fast ? lean_dec_kernel<R, true, true> : lean_dec_kernel<R, true, false>)
              : (fast ? lean_dec_kernel<R, false, true> : lean_dec_kernel<R, false, false>);
  launch_pdl(k, blocks, 32 * kLeanWPB, lean_dec_smem<R>(), s, g, st[0], st[1], st[2], sc[0],
             sc[1], sc[2], in, cls, P, f, t);
}
template <typename R>
void launch_lean_rload(bool fast, const LevelGeom<R> &g,
                       const std::array<const LeanW<R> *, 3> &st,
                       const std::array<const Stencil<R> *, 3> &sc, const R *cls, R *f,
                       cudaStream_t s) {
  const bool z3 = g.n[2] > 1;
  const LeanTiles t = lean_rtiles<R>(g.m[0], g.m[1], g.m[2], z3, fast);
  const unsigned blocks = unsigned((t.warps() + kLeanWPB - 1) / kLeanWPB);
  auto k = z3 ? (fast ? lean_rload_kernel<R, true, true> : lean_rload_kernel<R, true, false>)
              : (fast ? lean_rload_kernel<R, false, true> : lean_rload_kernel<R, false, false>);
  launch_pdl(k, blocks, 32 * kLeanWPB, 0, s, g, st[0], st[1], st[2], sc[0], sc[1], sc[2], cls, f,
             t);
}
template <typename R>
void launch_lean_rgpk(bool fast, const LevelGeom<R> &g,
                      const std::array<const LeanW<R> *, 3> &st, const R *coarse,
                      const R *cls, R *out, cudaStream_t s) {
  const bool z3 = g.n[2] > 1;
  const LeanTiles t = lean_gtiles<R>(g.m[0], g.m[1], g.m[2], z3);
  const unsigned blocks = unsigned((t.warps() + kLeanWPB - 1) / kLeanWPB);
  using K = void (*)(LevelGeom<R>, const LeanW<R> *, const LeanW<R> *, const LeanW<R> *,
                     const R *, const R *, R *, LeanTiles);
  K k;
  if (z3)
    k = cls ? (fast ? lean_rgpk_kernel<R, true, true, true> : lean_rgpk_kernel<R, true, true, false>)
            : (fast ? lean_rgpk_kernel<R, true, false, true>
                    : lean_rgpk_kernel<R, true, false, false>);
  else
    k = cls ? (fast ? lean_rgpk_kernel<R, false, true, true>
                    : lean_rgpk_kernel<R, false, true, false>)
            : (fast ? lean_rgpk_kernel<R, false, false, true>
                    : lean_rgpk_kernel<R, false, false, false>);
  launch_pdl(k, blocks, 32 * kLeanWPB, 0, s, g, st[0], st[1], st[2], coarse, cls, out, t);
}
template <typename R>
void launch_rl2(bool fast, const LevelGeom<R> &g,
                const std::array<const Stencil<R> *, 3> &st, const R *cls, R *f,
                cudaStream_t s) {
  constexpr int CY = pair_cy<R>();
  const dim3 grid = pair_grid(g, 30);
  auto k = fast ? rl2_kernel<R, CY, true> : rl2_kernel<R, CY, false>;
  k<<<grid, 256, rl2_smem<R, CY>(), s>>>(g, st[0], st[1], st[2], cls, f, grid.x, grid.y,
                                         grid.z);
}
template <typename R>
void launch_rg2(bool fast, const LevelGeom<R> &g, const R *coarse, const R *cls, R *out,
                cudaStream_t s) {
  constexpr int CY = pair_cy<R>();
  const dim3 grid = pair_grid(g, 32);
  auto k = fast ? rg2_kernel<R, CY, true> : rg2_kernel<R, CY, false>;
  k<<<grid, 256, rg2_smem<R, CY>(), s>>>(g, coarse, cls, out, grid.x, grid.y, grid.z);
}

// Batched Thomas along kernel dim kd of the m-lattice `g.m`.
//   FAST policy: warp-parallel affine scans (thomas_scan.cuh) along x and y;
//   exact policy: one thread per fiber -- smem-resident along x
//   (thomas.cuh), streaming along y; z streams in both (a z fiber strides
//   the whole lattice: staging whole fibers per CTA thrashes the TLB, the
//   streaming kernel keeps every CTA on the same planes).
template <typename R, uint32_t SEG>
void launch_scan_rows(const ThomasGeom<R> &t, uint64_t nf, R *f, Epi epi, const R *base,
                      R *out, cudaStream_t s) {
  const uint64_t blocks = std::min<uint64_t>((nf + 7) / 8, 148 * 8);
  thomas_scan_rows_kernel<R, SEG><<<unsigned(blocks), 256, scan_rows_smem<R>(t.m), s>>>(
      f, t, nf, epi, base, out);
}
template <typename R, uint32_t SEG>
void launch_scan_cols(const ThomasGeom<R> &t, uint64_t S, uint64_t inner, uint64_t ostride,
                      uint64_t nf, R *f, Epi epi, const R *base, R *out, cudaStream_t s) {
  thomas_scan_cols_kernel<R, SEG><<<unsigned((nf + 31) / 32), 256, scan_cols_smem<R>(t.m),
                                    s>>>(f, t, S, inner, ostride, nf, epi, base, out);
}
template <typename R>
bool try_scan(int kd, const ThomasGeom<R> &t, uint64_t S, uint64_t inner, uint64_t ostride,
              uint64_t nf, R *f, Epi epi, const R *base, R *out, cudaStream_t s) {
  const uint32_t seg = scan_seg(t.m);
  if (seg > 33)
    return false;
  if (kd == 0) {
    switch (seg) {
    case 1: launch_scan_rows<R, 1>(t, nf, f, epi, base, out, s); return true;
    case 3: launch_scan_rows<R, 3>(t, nf, f, epi, base, out, s); return true;
    case 5: launch_scan_rows<R, 5>(t, nf, f, epi, base, out, s); return true;
    case 7: case 9: launch_scan_rows<R, 9>(t, nf, f, epi, base, out, s); return true;
    case 11: case 13: case 15: case 17:
      launch_scan_rows<R, 17>(t, nf, f, epi, base, out, s); return true;
    default: launch_scan_rows<R, 33>(t, nf, f, epi, base, out, s); return true;
    }
  }
  if (scan_cols_smem<R>(t.m) > thomas_smem_limit<R>())
    return false;
  switch (seg) {
  case 1: launch_scan_cols<R, 1>(t, S, inner, ostride, nf, f, epi, base, out, s); return true;
  case 3: launch_scan_cols<R, 3>(t, S, inner, ostride, nf, f, epi, base, out, s); return true;
  case 5: launch_scan_cols<R, 5>(t, S, inner, ostride, nf, f, epi, base, out, s); return true;
  case 7: case 9:
    launch_scan_cols<R, 9>(t, S, inner, ostride, nf, f, epi, base, out, s); return true;
  case 11: case 13: case 15: case 17:
    launch_scan_cols<R, 17>(t, S, inner, ostride, nf, f, epi, base, out, s); return true;
  default:
    launch_scan_cols<R, 33>(t, S, inner, ostride, nf, f, epi, base, out, s); return true;
  }
}

template <typename R> constexpr size_t tf_limit() { return 224 * 1024; }

// small coarse lattices: one CTA solves every dimension (thomas_small_kernel)
#ifndef TS_SMEM_KB
#define TS_SMEM_KB 96
#endif
template <typename R> bool ts_fits(const LevelGeom<R> &g) {
  return g_thomas_small &&
         ts_smem<R>(g.coarse_nodes(), uint64_t(g.m[0]) + g.m[1] + g.m[2]) <= size_t(TS_SMEM_KB) * 1024;
}
template <typename R>
void launch_thomas_small(const LevelGeom<R> &g, const std::array<ThomasGeom<R>, 3> &t, R *f,
                         Epi epi, const R *base, R *out, cudaStream_t s) {
  launch_pdl(thomas_small_kernel<R>, 1, kTsThreads,
             ts_smem<R>(g.coarse_nodes(), uint64_t(g.m[0]) + g.m[1] + g.m[2]), s, f, t[0], t[1],
             t[2], g.m[0], g.m[1], g.m[2], g.refine, epi, base, out);
}

template <typename R, int DIM, int CH> auto tf_kernel() {
  return thomas_fiber_kernel<R, DIM, CH, 32>;
}
template <typename R, int DIM>
void (*tf_pick(int ch))(R *, ThomasLean<R>, uint64_t, uint32_t, uint32_t, Epi, const R *, R *) {
  switch (ch) {
  case 1: return tf_kernel<R, DIM, 1>();
  case 2: return tf_kernel<R, DIM, 2>();
  case 3: return tf_kernel<R, DIM, 3>();
  case 5: return tf_kernel<R, DIM, 5>();
  case 9: return tf_kernel<R, DIM, 9>();
  case 17: return tf_kernel<R, DIM, 17>();
  default: return tf_kernel<R, DIM, 33>();
  }
}
// the cluster kernel: cl CTAs of nw warps, chunk length 17 or 33
template <typename R, int DIM, int CH, int NW>
void (*tc_pick_cl(int cl))(R *, ThomasLean<R>, uint64_t, uint32_t, uint32_t, Epi, const R *,
                           R *) {
  if constexpr (TF_CL16 && NW == 8 && sizeof(R) == 8)
    if (cl == 16)
      return thomas_cluster_kernel<R, DIM, CH, 16, NW>;
  switch (cl) {
  case 1: return thomas_cluster_kernel<R, DIM, CH, 1, NW>;
  case 2: return thomas_cluster_kernel<R, DIM, CH, 2, NW>;
  case 4: return thomas_cluster_kernel<R, DIM, CH, 4, NW>;
  default: return thomas_cluster_kernel<R, DIM, CH, 8, NW>;
  }
}
template <typename R, int DIM>
void (*tc_pick(int ch, int cl, int nw))(R *, ThomasLean<R>, uint64_t, uint32_t, uint32_t, Epi,
                                        const R *, R *) {
  if constexpr (sizeof(R) == 8 || TF_NW8_F32)
    if (nw == 8)
      return ch <= 17 ? tc_pick_cl<R, DIM, 17, 8>(cl) : tc_pick_cl<R, DIM, 33, 8>(cl);
  return ch <= 17 ? tc_pick_cl<R, DIM, 17, 16>(cl) : tc_pick_cl<R, DIM, 33, 16>(cl);
}
template <typename R, int CH, int NW> size_t tc_smem_dim(int kd) {
  return kd == 0 ? tc_smem<R, 0, CH, NW>() : (kd == 1 ? tc_smem<R, 1, CH, NW>()
                                                       : tc_smem<R, 2, CH, NW>());
}
template <typename R> size_t tc_smem_of(int kd, int ch, int nw) {
  if (nw == 8)
    return ch <= 17 ? tc_smem_dim<R, 17, 8>(kd) : tc_smem_dim<R, 33, 8>(kd);
  return ch <= 17 ? tc_smem_dim<R, 17, 16>(kd) : tc_smem_dim<R, 33, 16>(kd);
}
// smem of the chunked-Thomas launch for a fiber length (either kernel)
template <typename R> size_t tf_launch_smem(int kd, uint32_t m) {
  return tf_clustered<R>(m, kd) ? tc_smem_of<R>(kd, tf_ch<R>(m, kd), tf_nw<R>(m, kd))
                            : tf_smem<R>(kd, m);
}
template <typename R>
void launch_tf(int kd, const ThomasLean<R> &tl, uint64_t nfib, uint32_t mx, uint32_t my,
               Epi epi, const R *base, R *out, R *f, cudaStream_t s) {
  const int ch = tf_ch<R>(tl.m, kd), cl = tf_cl<R>(tl.m, kd), nw = tf_nw<R>(tl.m, kd);
  const unsigned groups = unsigned((nfib + 31) / 32);
  if (tf_clustered<R>(tl.m, kd)) {
    auto k = kd == 0 ? tc_pick<R, 0>(ch, cl, nw)
                     : (kd == 1 ? tc_pick<R, 1>(ch, cl, nw) : tc_pick<R, 2>(ch, cl, nw));
    cudaLaunchConfig_t cfg = {};
    // persistent: as many clusters as are co-resident (queried once per
    // instantiation), each walking the 32-fiber groups
    static std::mutex mu;
    static std::map<const void *, int> resident;
    int nres = 0;
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = resident.find(reinterpret_cast<const void *>(k));
      if (it == resident.end()) {
        cudaLaunchConfig_t q = {};
        q.gridDim = dim3(unsigned(cl));
        q.blockDim = dim3(unsigned(32 * nw));
        q.dynamicSmemBytes = tc_smem_of<R>(kd, ch, nw);
        cudaLaunchAttribute qa[1];
        qa[0].id = cudaLaunchAttributeClusterDimension;
        qa[0].val.clusterDim.x = unsigned(cl);
        qa[0].val.clusterDim.y = 1;
        qa[0].val.clusterDim.z = 1;
        q.attrs = qa;
        q.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&nres, k, &q) != cudaSuccess || nres < 1) {
          cudaGetLastError();
          nres = 1;
        }
        resident[reinterpret_cast<const void *>(k)] = nres;
      } else {
        nres = it->second;
      }
    }
    cfg.gridDim = dim3(std::min<unsigned>(groups, unsigned(nres)) * unsigned(cl));
    cfg.blockDim = dim3(unsigned(32 * nw));
    cfg.dynamicSmemBytes = tc_smem_of<R>(kd, ch, nw);
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = unsigned(cl);
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, k, f, tl, nfib, mx, my, epi, base, out);
    return;
  }
  auto k = kd == 0 ? tf_pick<R, 0>(ch) : (kd == 1 ? tf_pick<R, 1>(ch) : tf_pick<R, 2>(ch));
  launch_pdl(k, groups, kTfThreads, tf_smem<R>(kd, tl.m), s, f, tl, nfib, mx, my, epi, base, out);
}
template <typename R> uint64_t tp_scratch_elems(mgrg_plan *p) {
  PlanT<R> &P = pt<R>(p);
  uint64_t need = 0;
  for (size_t l = 1; l < P.ttp.size(); ++l)
    for (int kd = 0; kd < 3; ++kd)
      if (P.ttp[l][kd].q) {
        const LevelGeom<R> &g = P.geom[l];
        const uint64_t nfib = g.coarse_nodes() / g.m[kd];
        need = std::max(need, 2 * nfib * P.ttp[l][kd].K);
      }
  return need;
}
template <typename R> void tp_bind_scratch(mgrg_plan *p) {
  PlanT<R> &P = pt<R>(p);
  for (size_t l = 1; l < P.ttp.size(); ++l)
    for (int kd = 0; kd < 3; ++kd)
      if (P.ttp[l][kd].q)
        P.ttp[l][kd].scratch = static_cast<R *>(p->d_ws) + p->offTP;
}
// Two-pass long-fiber solve: pass 1 (chunk summaries), carry scans, pass 2
// (chunk re-solve + epilogue); E / S scratch = 2 * nfib * K elements.
template <typename R>
void launch_tp(int kd, const ThomasTP<R> &tp, R *scratch, uint64_t nfib, uint32_t mx,
               uint32_t my, Epi epi, const R *base, R *out, R *f, cudaStream_t s) {
  R *E = scratch, *S = scratch + nfib * tp.K;
  const dim3 grid(unsigned((nfib + 32 * kTpWarps - 1) / (32 * kTpWarps)), tp.K);
  auto k1 = kd == 1 ? tp_pass1_kernel<R, 1> : tp_pass1_kernel<R, 2>;
  launch_pdl(k1, grid, 32 * kTpWarps, 0, s, static_cast<const R *>(f), tp, nfib, mx, my, E, S);
  launch_pdl(tp_carry_kernel<R>, unsigned((nfib + 31) / 32), 32 * kTcWarps, 0, s, tp, nfib, E,
             S);
  auto k2 = kd == 1 ? tp_pass2_kernel<R, 1> : tp_pass2_kernel<R, 2>;
  launch_pdl(k2, grid, 32 * kTpWarps, 0, s, f, tp, nfib, mx, my, static_cast<const R *>(E),
             static_cast<const R *>(S), epi, base, out);
}
template <typename R> void set_tf_attrs() {
  const int lim = int(tf_limit<R>());
  for (int ch : {1, 2, 3, 5, 9, 17, 33}) {
    cudaFuncSetAttribute(tf_pick<R, 0>(ch), cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
    cudaFuncSetAttribute(tf_pick<R, 1>(ch), cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
    cudaFuncSetAttribute(tf_pick<R, 2>(ch), cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  }
  if (TF_CL16)
    for (int ch : {17, 33})
      for (auto k : {tc_pick<R, 0>(ch, 16, 8), tc_pick<R, 1>(ch, 16, 8),
                     tc_pick<R, 2>(ch, 16, 8)})
        cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int nw : {8, 16})
    for (int ch : {17, 33})
      for (int cl : {1, 2, 4, 8, 16}) {
        cudaFuncSetAttribute(tc_pick<R, 0>(ch, cl, nw),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
        cudaFuncSetAttribute(tc_pick<R, 1>(ch, cl, nw),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
        cudaFuncSetAttribute(tc_pick<R, 2>(ch, cl, nw),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
      }
}

template <typename R>
void launch_thomas(bool fast, const LevelGeom<R> &g, const ThomasGeom<R> &t,
                   const ThomasLean<R> &tl, int kd, R *f, Epi epi, const R *base, R *out,
                   cudaStream_t s, const ThomasTP<R> *tp = nullptr,
                   uint64_t *extra_launches = nullptr) {
  const uint64_t mx = g.m[0], my = g.m[1], mz = g.m[2];
  if (fast && kd != 0 && tp && tp->q && tp->scratch && tp->m >= uint32_t(g_tp_min)) {
    const uint64_t nfib = kd == 0 ? my * mz : (kd == 1 ? mx * mz : mx * my);
    launch_tp<R>(kd, *tp, tp->scratch, nfib, uint32_t(mx), uint32_t(my), epi, base, out, f, s);
    if (extra_launches)
      *extra_launches += 2; // three kernels for one counted solve
    return;
  }
  if (fast && tl.tab && tf_ch<R>(tl.m, kd) && tf_launch_smem<R>(kd, tl.m) <= tf_limit<R>() &&
      g_thomas_fiber) {
    const uint64_t nfib = kd == 0 ? my * mz : (kd == 1 ? mx * mz : mx * my);
    launch_tf<R>(kd, tl, nfib, uint32_t(mx), uint32_t(my), epi, base, out, f, s);
    return;
  }
  if (!fast && g_thomas_exact && (kd == 0 || g_thomas_exact > 1) && te_fits<R>(kd, t.m) &&
      (reinterpret_cast<uintptr_t>(f) & 15) == 0) {
    // exact order, fibers resident in shared memory (thomas_exact.cuh); x
    // fibers only by default: for y / z the thread-per-fiber streaming kernel
    // measured faster (0.48 / 0.87 ms vs 0.73 / 1.26 ms at 1025^3 f32)
    const uint64_t nfib = kd == 0 ? my * mz : (kd == 1 ? mx * mz : mx * my);
    const unsigned blocks = unsigned((nfib + te_nf<R>() - 1) / te_nf<R>());
    auto k = kd == 0 ? thomas_exact_kernel<R, 0>
                     : (kd == 1 ? thomas_exact_kernel<R, 1> : thomas_exact_kernel<R, 2>);
    launch_pdl(k, blocks, kTeThreads, te_smem<R>(kd, t.m), s, f, t, nfib, uint32_t(mx),
               uint32_t(my), epi, base, out);
    return;
  }
  if (kd == 0) {
    const uint64_t nf = my * mz;
    if (fast && try_scan<R>(0, t, 1, 1, 0, nf, f, epi, base, out, s))
      return;
    if (!fast && thomas_resident_fits<R>(t.m)) {
      thomas_rows_kernel<R, false><<<unsigned((nf + kThomasFibers - 1) / kThomasFibers),
                                     kThomasFibers, thomas_rows_smem<R>(t.m), s>>>(
          f, t, nf, epi, base, out);
      return;
    }
    const uint64_t warps = (nf + 31) / 32;
    thomas_x_kernel<R><<<unsigned((warps + 3) / 4), 128, 0, s>>>(f, t, nf, epi, base,
                                                                 out);
  } else {
    const uint64_t S = kd == 1 ? mx : mx * my;
    const uint64_t ostride = kd == 1 ? mx * my : mx; // the remaining dim
    const uint64_t nf = mx * (kd == 1 ? mz : my);
    if (fast && kd == 1 && try_scan<R>(1, t, S, mx, mx * my, nf, f, epi, base, out, s))
      return;
    launch_pdl(thomas_strided_kernel<R, 8>, unsigned((nf + 127) / 128), 128, 0, s, f, t, S,
               uint32_t(mx), ostride, nf, epi, base, out);
  }
}

template <typename R, uint32_t SEG> void set_scan_attrs(int lim) {
  cudaFuncSetAttribute(thomas_scan_rows_kernel<R, SEG>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  cudaFuncSetAttribute(thomas_scan_cols_kernel<R, SEG>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
}
template <typename R> void set_thomas_attrs() {
  const int lim = int(thomas_smem_limit<R>());
  set_scan_attrs<R, 1>(lim);
  set_scan_attrs<R, 3>(lim);
  set_scan_attrs<R, 5>(lim);
  set_scan_attrs<R, 9>(lim);
  set_scan_attrs<R, 17>(lim);
  set_scan_attrs<R, 33>(lim);
  cudaFuncSetAttribute(thomas_rows_kernel<R, false>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  cudaFuncSetAttribute(thomas_rows_kernel<R, true>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  cudaFuncSetAttribute(thomas_cols_kernel<R, false>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  cudaFuncSetAttribute(thomas_cols_kernel<R, true>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  set_tf_attrs<R>();
  for (auto k : {thomas_exact_kernel<R, 0>, thomas_exact_kernel<R, 1>, thomas_exact_kernel<R, 2>})
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 74 * 1024);
  cudaFuncSetAttribute(thomas_small_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       TS_SMEM_KB * 1024);
}

template <typename R> R *ws(mgrg_plan *p, uint64_t off) {
  return static_cast<R *>(p->d_ws) + off;
}
// Buffer holding the packed level-j array, 1 <= j <= L-1 (ping-pong A/B).
template <typename R> R *level_buf(mgrg_plan *p, int j) {
  return ((p->H.L - 1 - j) % 2 == 0) ? ws<R>(p, p->offA) : ws<R>(p, p->offB);
}

// Launch bookkeeping: counts every kernel of a call and, when profiling is
// on, brackets each launch with CUDA events on the launch stream so the
// caller can read per-kernel device time next to the algorithmic bytes.
struct Recorder {
  mgrg_plan *p;
  cudaStream_t s;
  uint64_t launches = 0;
  bool active = false; // the current launch is bracketed by events
  mgrg_status begin(int kind, int level, uint64_t bytes);
  mgrg_status end();
};

mgrg_status Recorder::begin(int kind, int level, uint64_t bytes) {
  ++launches;
  active = p->profiling && level >= p->prof_min_level;
  if (!active)
    return MGRG_OK;
  if (p->prof_used + 2 > p->event_pool.size()) {
    for (int i = 0; i < 64; ++i) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreate(&e));
      p->event_pool.push_back(e);
    }
  }
  mgrg_plan::Prof pr{kind, level, bytes, p->event_pool[p->prof_used],
                     p->event_pool[p->prof_used + 1]};
  p->prof_used += 2;
  CUDA_TRY(prof_record(pr.e0, s));
  p->prof.push_back(pr);
  return MGRG_OK;
}

mgrg_status Recorder::end() {
  if (!active)
    return MGRG_OK;
  CUDA_TRY(prof_record(p->prof.back().e1, s));
  return MGRG_OK;
}

// ---- 4-D levels (gen4.cuh) -------------------------------------------------

inline unsigned gen_blocks(uint64_t n) { return unsigned((n + 255) / 256); }

// Thomas along dim d of the compact coarse lattice with the 3-D family's
// exact-order kernels: x fibers resident in shared memory, the others one
// thread per fiber with consecutive threads on consecutive inner nodes
template <typename R> void gen_launch_thomas(const Gen4Geom<R> &g, int d, R *f, cudaStream_t s) {
  const ThomasGeom<R> t{g.th[d], g.tf[d], g.ti[d], g.m[d]};
  const uint64_t nfib = g.coarse_nodes() / g.m[d];
  if (d == 0 && te_fits<R>(0, t.m) && (reinterpret_cast<uintptr_t>(f) & 15) == 0) {
    thomas_exact_kernel<R, 0><<<unsigned((nfib + te_nf<R>() - 1) / te_nf<R>()), kTeThreads,
                                te_smem<R>(0, t.m), s>>>(f, t, nfib, g.m[0], g.m[1], Epi::none,
                                                         nullptr, nullptr);
    return;
  }
  uint64_t inner = 1;
  for (int k = 0; k < d; ++k)
    inner *= g.m[k];
  thomas_strided_kernel<R><<<unsigned((nfib + 127) / 128), 128, 0, s>>>(
      f, t, inner, inner, inner * g.m[d], nfib, Epi::none, nullptr, nullptr);
}

// R*M along every refining dimension, dims ascending (masstrans_dim0 then
// masstrans_later, refactor.hpp:251-346), ping-pong between W and W2;
// returns the buffer holding the load vector on the coarse lattice
template <typename R>
R *gen_mass_all(mgrg_plan *p, const Gen4Geom<R> &g, int l, Recorder &rec, cudaStream_t s,
                mgrg_status &st) {
  R *cur = ws<R>(p, p->offW), *oth = ws<R>(p, p->offW2);
  uint32_t e[kGenDims] = {g.n[0], g.n[1], g.n[2], g.n[3]};
  for (int d = 0; d < kGenDims; ++d) {
    if (!(g.m[d] < g.n[d]))
      continue;
    uint64_t out = 1;
    for (int k = 0; k < kGenDims; ++k)
      out *= k == d ? g.m[d] : e[k];
    if ((st = rec.begin(MGRG_K_DEC_LEVEL, l, 0)))
      return nullptr;
    gen_mass_kernel<R><<<gen_blocks(out), 256, 0, s>>>(g, d, make_uint4(e[0], e[1], e[2], e[3]),
                                                       cur, oth);
    if ((st = rec.end()))
      return nullptr;
    e[d] = g.m[d];
    std::swap(cur, oth);
  }
  // Thomas along every refining dimension, in place on the coarse lattice
  for (int d = 0; d < kGenDims; ++d) {
    if (!(g.m[d] < g.n[d]))
      continue;
    if ((st = rec.begin(MGRG_K_THOMAS_X + std::min(d, 2), l, 0)))
      return nullptr;
    gen_launch_thomas<R>(g, d, cur, s);
    if ((st = rec.end()))
      return nullptr;
  }
  return cur;
}

template <typename R>
mgrg_status run_gen_decompose(mgrg_plan *p, const R *d_in, R *d_cls, cudaStream_t s) {
  PlanT<R> &P = pt<R>(p);
  const int L = p->H.L;
  Recorder rec{p, s};
  mgrg_status st = MGRG_OK;
  for (int l = L; l >= 1; --l) {
    const Gen4Geom<R> &g = P.g4[l];
    const R *a = l == L ? d_in : level_buf<R>(p, l);
    R *Pout = l == 1 ? d_cls : level_buf<R>(p, l - 1);
    R *cls = d_cls + p->nodes[l - 1];
    if ((st = rec.begin(MGRG_K_DEC_LEVEL, l, 0)))
      return st;
    gen_coef_kernel<R><<<gen_blocks(g.nodes()), 256, 0, s>>>(g, a, ws<R>(p, p->offW), cls);
    if ((st = rec.end()))
      return st;
    R *z = gen_mass_all<R>(p, g, l, rec, s, st);
    if (st)
      return st;
    if ((st = rec.begin(MGRG_K_DEC_LEVEL, l, 0)))
      return st;
    gen_apply_kernel<R><<<gen_blocks(g.coarse_nodes()), 256, 0, s>>>(g, a, z, Pout);
    if ((st = rec.end()))
      return st;
  }
  CUDA_TRY(cudaGetLastError());
  p->last_launches = rec.launches;
  return MGRG_OK;
}

template <typename R>
mgrg_status run_gen_recompose(mgrg_plan *p, const R *d_cls, int k, R *d_out, cudaStream_t s) {
  PlanT<R> &P = pt<R>(p);
  const int L = p->H.L;
  Recorder rec{p, s};
  mgrg_status st = MGRG_OK;
  for (int l = 1; l <= L; ++l) {
    const Gen4Geom<R> &g = P.g4[l];
    const R *prev = l == 1 ? d_cls : level_buf<R>(p, l - 1);
    R *out = l == L ? d_out : level_buf<R>(p, l);
    const R *cls = l <= k ? d_cls + p->nodes[l - 1] : nullptr;
    const R *cz = prev; // classes above k are zero: z = +0, a' = a_{l-1} exactly
    if (cls) {
      if ((st = rec.begin(MGRG_K_REC_LOAD, l, 0)))
        return st;
      gen_load_kernel<R><<<gen_blocks(g.nodes()), 256, 0, s>>>(g, cls, ws<R>(p, p->offW));
      if ((st = rec.end()))
        return st;
      R *z = gen_mass_all<R>(p, g, l, rec, s, st);
      if (st)
        return st;
      if ((st = rec.begin(MGRG_K_REC_LOAD, l, 0)))
        return st;
      gen_unapply_kernel<R><<<gen_blocks(g.coarse_nodes()), 256, 0, s>>>(g.coarse_nodes(), prev,
                                                                          z);
      if ((st = rec.end()))
        return st;
      cz = z;
    }
    if ((st = rec.begin(MGRG_K_REC_GPK, l, 0)))
      return st;
    gen_rgpk_kernel<R><<<gen_blocks(g.nodes()), 256, 0, s>>>(g, cz, cls, out);
    if ((st = rec.end()))
      return st;
  }
  CUDA_TRY(cudaGetLastError());
  p->last_launches = rec.launches;
  return MGRG_OK;
}

template <typename R>
mgrg_status run_decompose(mgrg_plan *p, const R *d_in, R *d_cls, cudaStream_t s,
                          bool top_done = false) {
  if (p->gen)
    return run_gen_decompose<R>(p, d_in, d_cls, s);
  PlanT<R> &P = pt<R>(p);
  const int L = p->H.L;
  R *F = ws<R>(p, p->offF);
  Recorder rec{p, s};
  const uint64_t es = sizeof(R);
  for (int l = L; l >= 1; --l) {
    const LevelGeom<R> &g = P.geom[l];
    const uint64_t Fn = g.nodes(), Cn = g.coarse_nodes();
    const R *a = l == L ? d_in : level_buf<R>(p, l);
    R *Pout = l == 1 ? d_cls : level_buf<R>(p, l - 1);
    R *cls = d_cls + p->nodes[l - 1];
    // read F; write class (F-C) + packed coarse (C) + load vector (C)
    if (!(top_done && l == L)) {
    if (mgrg_status st = rec.begin(MGRG_K_DEC_LEVEL, l, es * (2 * Fn + Cn)))
      return st;
    // dec4 stages rows with 16-byte copies: the level array must be 16-byte
    // aligned (workspace levels are; a caller's input may not be)
    const bool al16 = (reinterpret_cast<uintptr_t>(a) & 15) == 0;
    // the lean kernel stages 16-byte aligned row supersets of the level array
    if (p->lean && al16 && lean_level(g))
      launch_lean_dec<R>(p->fast, g, P.lean[l], P.sten[l], a, cls, Pout, F, s);
    else if (p->pair_path && al16)
      launch_dec4<R>(p->fast, g, P.sten[l], a, cls, Pout, F, s);
    else if (p->tile == TileKind::t32x8)
      launch_dec_level<R, 32, 8>(g, a, cls, Pout, F, p->zchunk, s);
    else
      launch_dec_level<R, 128, 1>(g, a, cls, Pout, F, p->zchunk, s);
    if (mgrg_status st = rec.end())
      return st;
    }
    if (p->fast && ts_fits<R>(g)) {
      // all solves + apply in one launch (small coarse lattice)
      if (mgrg_status st = rec.begin(MGRG_K_THOMAS_X, l, es * Cn * 3))
        return st;
      launch_thomas_small<R>(g, P.thom[l], F, Epi::add, Pout, Pout, s);
      if (mgrg_status st = rec.end())
        return st;
      continue;
    }
    for (int i = 0; i < p->nrefine; ++i) {
      const int kd = p->refine_dims[i];
      const bool last = i == p->nrefine - 1;
      // f in + z out; the fused apply also reads the packed coarse values
      if (mgrg_status st = rec.begin(MGRG_K_THOMAS_X + kd, l, es * Cn * (last ? 3 : 2)))
        return st;
      launch_thomas<R>(p->fast, g, P.thom[l][kd], P.tlean[l][kd], kd, F,
                       last ? Epi::add : Epi::none, Pout, Pout, s, &P.ttp[l][kd],
                       &rec.launches);
      if (mgrg_status st = rec.end())
        return st;
    }
  }
  CUDA_TRY(cudaGetLastError());
  p->last_launches = rec.launches;
  return MGRG_OK;
}

template <typename R>
mgrg_status run_recompose(mgrg_plan *p, const R *d_cls, int k, R *d_out,
                          cudaStream_t s, int lmax = -1) {
  if (p->gen)
    return run_gen_recompose<R>(p, d_cls, k, d_out, s);
  PlanT<R> &P = pt<R>(p);
  const int L = p->H.L;
  R *F = ws<R>(p, p->offF);
  Recorder rec{p, s};
  const uint64_t es = sizeof(R);
  for (int l = 1; l <= (lmax < 0 ? L : lmax); ++l) {
    const LevelGeom<R> &g = P.geom[l];
    const uint64_t Fn = g.nodes(), Cn = g.coarse_nodes();
    const R *prev = l == 1 ? d_cls : level_buf<R>(p, l - 1);
    R *out = l == L ? d_out : level_buf<R>(p, l);
    const R *cls = d_cls + p->nodes[l - 1];
    if (l <= k) {
      // read class (F-C); write load vector (C)
      if (mgrg_status st = rec.begin(MGRG_K_REC_LOAD, l, es * Fn))
        return st;
      if (p->lean && lean_level(g))
        launch_lean_rload<R>(p->fast, g, P.lean[l], P.sten[l], cls, F, s);
      else if (p->pair_path)
        launch_rl2<R>(p->fast, g, P.sten[l], cls, F, s);
      else if (p->tile == TileKind::t32x8)
        launch_rec_load<R, 32, 8>(g, cls, F, p->zchunk, s);
      else
        launch_rec_load<R, 128, 1>(g, cls, F, p->zchunk, s);
      if (mgrg_status st = rec.end())
        return st;
      const bool small = p->fast && ts_fits<R>(g);
      if (small) {
        if (mgrg_status st = rec.begin(MGRG_K_THOMAS_X, l, es * Cn * 3))
          return st;
        launch_thomas_small<R>(g, P.thom[l], F, Epi::sub, prev, F, s);
        if (mgrg_status st = rec.end())
          return st;
      }
      for (int i = 0; i < (small ? 0 : p->nrefine); ++i) {
        const int kd = p->refine_dims[i];
        const bool last = i == p->nrefine - 1;
        if (mgrg_status st = rec.begin(MGRG_K_THOMAS_X + kd, l, es * Cn * (last ? 3 : 2)))
          return st;
        launch_thomas<R>(p->fast, g, P.thom[l][kd], P.tlean[l][kd], kd, F,
                         last ? Epi::sub : Epi::none, prev, F, s, &P.ttp[l][kd],
                         &rec.launches);
        if (mgrg_status st = rec.end())
          return st;
      }
      // read coarse' (C) + class (F-C); write the level array (F)
      if (mgrg_status st = rec.begin(MGRG_K_REC_GPK, l, es * 2 * Fn))
        return st;
      if (p->lean && lean_level(g) && lean_out_ok<R>(out))
        launch_lean_rgpk<R>(p->fast, g, P.lean[l], F, cls, out, s);
      else if (p->pair_path)
        launch_rg2<R>(p->fast, g, F, cls, out, s);
      else if (p->tile == TileKind::t32x8)
        launch_rec_gpk<R, 32, 8>(g, F, cls, out, p->zchunk, s);
      else
        launch_rec_gpk<R, 128, 1>(g, F, cls, out, p->zchunk, s);
    } else {
      // classes above classes_used are zero: f = 0, z = +0 exactly, so the
      // coarse values are a_{l-1} unchanged and the fine ones interp + 0.
      if (mgrg_status st = rec.begin(MGRG_K_REC_GPK, l, es * (Fn + Cn)))
        return st;
      if (p->lean && lean_level(g) && lean_out_ok<R>(out))
        launch_lean_rgpk<R>(p->fast, g, P.lean[l], prev, nullptr, out, s);
      else if (p->pair_path)
        launch_rg2<R>(p->fast, g, prev, nullptr, out, s);
      else if (p->tile == TileKind::t32x8)
        launch_rec_gpk<R, 32, 8>(g, prev, nullptr, out, p->zchunk, s);
      else
        launch_rec_gpk<R, 128, 1>(g, prev, nullptr, out, p->zchunk, s);
    }
    if (mgrg_status st = rec.end())
      return st;
  }
  CUDA_TRY(cudaGetLastError());
  p->last_launches = rec.launches;
  return MGRG_OK;
}

mgrg_status check_plan(const mgrg_plan *p) {
  if (!p)
    return fail(MGRG_INVALID_ARGUMENT, "null plan");
  return MGRG_OK;
}

} // namespace

extern "C" {

const char *mgrg_version(void) { return "mgrg-b200 0.1 (sm_100a)"; }

const char *mgrg_last_error(void) { return g_last_error.c_str(); }

const char *mgrg_status_name(mgrg_status st) {
  switch (st) {
  case MGRG_OK: return "Ok";
  case MGRG_INVALID_GRID: return "InvalidGrid";
  case MGRG_INVALID_LEVEL: return "InvalidLevel";
  case MGRG_SHAPE_ERROR: return "ShapeError";
  case MGRG_INVALID_FUSION: return "InvalidFusion";
  case MGRG_SINGULAR_SYSTEM: return "SingularSystem";
  case MGRG_TOO_MANY_WORKERS: return "TooManyWorkers";
  case MGRG_WORKER_FAILURE: return "WorkerFailure";
  case MGRG_CORRUPT_FILE: return "CorruptFile";
  case MGRG_MISSING_CLASS: return "MissingClass";
  case MGRG_INVALID_BOUND: return "InvalidBound";
  case MGRG_IO_ERROR: return "IoError";
  case MGRG_CUDA_ERROR: return "CudaError";
  case MGRG_NCCL_ERROR: return "NcclError";
  case MGRG_UNSUPPORTED: return "Unsupported";
  case MGRG_INVALID_ARGUMENT: return "InvalidArgument";
  case MGRG_OUT_OF_MEMORY: return "OutOfMemory";
  }
  return "Unknown";
}

mgrg_status mgrg_plan_create(const mgrg_grid_desc *desc, mgrg_plan **out) {
  g_last_error.clear();
  if (!desc || !out)
    return fail(MGRG_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (desc->dtype != MGRG_F32 && desc->dtype != MGRG_F64)
    return fail(MGRG_INVALID_ARGUMENT, "dtype must be MGRG_F32 or MGRG_F64");
  std::unique_ptr<mgrg_plan> p(new mgrg_plan());
  p->device = desc->device;
  p->dtype = desc->dtype;
  p->esize = desc->dtype;
  if (mgrg_status st = build_hierarchy(*desc, p->H))
    return st;
  const Hierarchy &H = p->H;
  const int nd = H.nd, L = H.L;
  auto al = [](uint64_t n) { return (n + 63) & ~uint64_t(63); };
  if (nd == 4) {
    // 4-D: generic per-pass kernels (gen4.cuh); both policies bit-exact
    p->gen = true;
    p->fast = (desc->flags & MGRG_FLAG_FAST) != 0;
    p->kext.assign(L + 1, {1, 1, 1});
    p->nodes.assign(L + 1, 1);
    for (int l = 0; l <= L; ++l)
      for (int d = 0; d < nd; ++d)
        p->nodes[l] *= H.ext[l][d];
    DeviceGuard guard(p->device);
    mgrg_status st = p->dtype == MGRG_F32 ? upload_geometry_gen<float>(p.get())
                                          : upload_geometry_gen<double>(p.get());
    if (st)
      return st;
    // workspace: A = N_{L-1}, B = N_{L-2} (level ping-pong), W, W2 = N_L
    const uint64_t nA = p->nodes[L - 1], nB = L >= 2 ? p->nodes[L - 2] : 1;
    p->offA = 0;
    p->offB = al(nA);
    p->offW = p->offB + al(nB);
    p->offW2 = p->offW + al(p->nodes[L]);
    p->offF = p->offW2;
    p->ws_bytes = (p->offW2 + al(p->nodes[L])) * p->esize;
    cudaError_t e = cudaMalloc(&p->d_ws, p->ws_bytes);
    if (e != cudaSuccess) {
      cudaFree(p->d_geom);
      return fail(e == cudaErrorMemoryAllocation ? MGRG_OUT_OF_MEMORY : MGRG_CUDA_ERROR,
                  std::string("workspace allocation: ") + cudaGetErrorString(e));
    }
    if (p->dtype == MGRG_F32)
      set_thomas_attrs<float>();
    else
      set_thomas_attrs<double>();
    *out = p.release();
    return MGRG_OK;
  }
  // kernel dims: user dims in order, padded to 3
  for (int kd = 0; kd < 3; ++kd)
    p->kmap[kd] = kd < nd ? kd : -1;
  p->kext.assign(L + 1, {1, 1, 1});
  p->nodes.assign(L + 1, 1);
  for (int l = 0; l <= L; ++l)
    for (int kd = 0; kd < 3; ++kd) {
      const int ud = p->kmap[kd];
      p->kext[l][kd] = ud < 0 ? 1 : uint32_t(H.ext[l][ud]);
      p->nodes[l] *= p->kext[l][kd];
    }
  p->refine = 0;
  p->nrefine = 0;
  for (int kd = 0; kd < 3; ++kd)
    if (p->kext[L - 1][kd] < p->kext[L][kd]) {
      p->refine |= 1u << kd;
      p->refine_dims[p->nrefine++] = kd;
    }
  p->tile = nd == 1 ? TileKind::t128x1 : TileKind::t32x8;
  p->pair_path = (p->refine & 3u) == 3u;
  p->fast = (desc->flags & MGRG_FLAG_FAST) != 0;
  if (knob("MGRG_GENERIC", 0) != 0)
    p->pair_path = false;
  {
    // lean family: x, y (and z) refine; used on every level whose extents
    // are all odd (coarse = even positions), see lean_level()
    p->lean = p->refine == 7u || (p->refine == 3u && p->kext[L][2] == 1);
    p->lean = p->lean && knob("MGRG_LEAN", 1) != 0;
    // the lean kernels index the level array and class buffer with 32-bit
    // element offsets
    p->lean = p->lean && p->nodes[L] < (uint64_t(1) << 32);
  }
  p->zchunk = nd == 3 ? 32 : 1;
  if (nd == 3 && knob("MGRG_ZCHUNK", 0) > 0)
    p->zchunk = uint32_t(knob("MGRG_ZCHUNK", 0));

  DeviceGuard guard(p->device);
  mgrg_status st = p->dtype == MGRG_F32 ? upload_geometry<float>(p.get())
                                        : upload_geometry<double>(p.get());
  if (st)
    return st;
  // workspace: A = N_{L-1}, B = N_{L-2}, F = N_{L-1}
  const uint64_t nA = p->nodes[L - 1];
  const uint64_t nB = L >= 2 ? p->nodes[L - 2] : 1;
  p->offA = 0;
  p->offB = al(nA);
  p->offF = p->offB + al(nB);
  // two-pass long-fiber Thomas scratch: the largest 2 * fibers * chunks
  const uint64_t nTP = p->dtype == MGRG_F32 ? tp_scratch_elems<float>(p.get())
                                            : tp_scratch_elems<double>(p.get());
  p->offTP = p->offF + al(nA);
  p->ws_bytes = (p->offTP + al(nTP)) * p->esize;
  cudaError_t e = cudaMalloc(&p->d_ws, p->ws_bytes);
  if (e != cudaSuccess) {
    cudaFree(p->d_geom);
    return fail(e == cudaErrorMemoryAllocation ? MGRG_OUT_OF_MEMORY : MGRG_CUDA_ERROR,
                std::string("workspace allocation: ") + cudaGetErrorString(e));
  }
  if (nTP) {
    if (p->dtype == MGRG_F32)
      tp_bind_scratch<float>(p.get());
    else
      tp_bind_scratch<double>(p.get());
  }
  if (p->dtype == MGRG_F32) {
    set_smem_attrs<float, 32, 8>();
    set_smem_attrs<float, 128, 1>();
    set_pair_attrs<float, pair_cy<float>()>();
    set_thomas_attrs<float>();
  } else {
    set_smem_attrs<double, 32, 8>();
    set_smem_attrs<double, 128, 1>();
    set_pair_attrs<double, pair_cy<double>()>();
    set_thomas_attrs<double>();
  }
  CUDA_TRY(cudaGetLastError());
  *out = p.release();
  return MGRG_OK;
}

mgrg_status mgrg_plan_destroy(mgrg_plan *p) {
  if (!p)
    return MGRG_OK;
  {
    DeviceGuard guard(p->device);
    p->xfer.reset(); // joins the download worker before its stream goes
    for (cudaEvent_t e : p->event_pool)
      cudaEventDestroy(e);
    cudaFree(p->d_geom);
    cudaFree(p->d_ws);
    cudaFree(p->d_stage);
    if (p->own_stream)
      cudaStreamDestroy(p->own_stream);
    for (cudaStream_t q : {p->s_in, p->s_out})
      if (q)
        cudaStreamDestroy(q);
    for (int i = 0; i < 16; ++i) {
      if (p->ev_in[i])
        cudaEventDestroy(p->ev_in[i]);
      if (p->ev_dec[i])
        cudaEventDestroy(p->ev_dec[i]);
    }
    if (p->ev_done)
      cudaEventDestroy(p->ev_done);
    for (auto &gr : p->graph_cache)
      cudaGraphExecDestroy(gr.exec);
    if (p->graph_stream)
      cudaStreamDestroy(p->graph_stream);
    for (cudaEvent_t e : p->graph_ev)
      if (e)
        cudaEventDestroy(e);
  }
  delete p;
  return MGRG_OK;
}

mgrg_status mgrg_plan_levels(const mgrg_plan *p, int32_t *levels) {
  if (mgrg_status st = check_plan(p))
    return st;
  if (!levels)
    return fail(MGRG_INVALID_ARGUMENT, "null output");
  *levels = p->H.L;
  return MGRG_OK;
}

mgrg_status mgrg_plan_class_offsets(const mgrg_plan *p, uint64_t *offsets) {
  if (mgrg_status st = check_plan(p))
    return st;
  if (!offsets)
    return fail(MGRG_INVALID_ARGUMENT, "null output");
  offsets[0] = 0;
  for (int l = 0; l <= p->H.L; ++l)
    offsets[l + 1] = p->nodes[l];
  return MGRG_OK;
}

mgrg_status mgrg_plan_level_shape(const mgrg_plan *p, int32_t level,
                                  uint64_t *extents) {
  if (mgrg_status st = check_plan(p))
    return st;
  if (level < 0 || level > p->H.L)
    return fail(MGRG_INVALID_LEVEL, "level " + std::to_string(level) +
                                        " outside [0, " + std::to_string(p->H.L) + "]");
  for (int d = 0; d < p->H.nd; ++d)
    extents[d] = p->H.ext[level][d];
  return MGRG_OK;
}

mgrg_status mgrg_plan_sizes(const mgrg_plan *p, uint64_t *n, uint64_t *wsb) {
  if (mgrg_status st = check_plan(p))
    return st;
  if (n)
    *n = p->nodes[p->H.L];
  if (wsb)
    *wsb = p->ws_bytes + p->geom_bytes;
  return MGRG_OK;
}

mgrg_status mgrg_plan_last_launches(const mgrg_plan *p, uint64_t *launches) {
  if (mgrg_status st = check_plan(p))
    return st;
  *launches = p->last_launches;
  return MGRG_OK;
}

mgrg_status mgrg_plan_set_profiling(mgrg_plan *p, int32_t enable) {
  if (mgrg_status st = check_plan(p))
    return st;
  p->profiling = enable != 0;
  // enable < 0: only the top -enable levels (fewer events in a timed loop)
  p->prof_min_level = enable < 0 ? p->H.L + 1 + enable : 0;
  return MGRG_OK;
}

mgrg_status mgrg_plan_profile_reset(mgrg_plan *p) {
  if (mgrg_status st = check_plan(p))
    return st;
  p->prof.clear();
  p->prof_used = 0;
  return MGRG_OK;
}

mgrg_status mgrg_plan_profile_read(mgrg_plan *p, uint64_t cap, int32_t *kinds,
                                   int32_t *levels, float *ms, uint64_t *bytes,
                                   uint64_t *count) {
  if (mgrg_status st = check_plan(p))
    return st;
  DeviceGuard guard(p->device);
  if (count)
    *count = p->prof.size();
  // (a device sync, not an event sync: events recorded by replayed graph
  // nodes cannot be host-synchronized)
  if (!p->prof.empty()) {
    DeviceGuard guard(p->device);
    CUDA_TRY(cudaDeviceSynchronize());
  }
  for (uint64_t i = 0; i < p->prof.size() && i < cap; ++i) {
    const auto &pr = p->prof[i];
    if (kinds)
      kinds[i] = pr.kind;
    if (levels)
      levels[i] = pr.level;
    if (bytes)
      bytes[i] = pr.bytes;
    if (ms) {
      float t = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&t, pr.e0, pr.e1));
      ms[i] = t;
    }
  }
  return MGRG_OK;
}

} // extern "C"

namespace {
constexpr size_t kGraphCache = 8;

// Run `body` (which launches the level loop on the stream it is given) as a
// replayed CUDA graph: captured once per (op, a, b, k) on the plan's graph
// stream -- the caller's stream may be the legacy default stream, which
// cannot be captured -- and launched there between two event hand-offs.
template <typename Body>
mgrg_status run_graphed(mgrg_plan *p, int op, const void *a, void *b, int32_t k,
                        cudaStream_t s, Body body) {
  if (!p->graph_stream) {
    CUDA_TRY(cudaStreamCreateWithFlags(&p->graph_stream, cudaStreamNonBlocking));
    for (cudaEvent_t &e : p->graph_ev)
      CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  auto &cache = p->graph_cache;
  size_t hit = cache.size();
  for (size_t i = 0; i < cache.size(); ++i)
    if (cache[i].op == op && cache[i].a == a && cache[i].b == b && cache[i].k == k)
      hit = i;
  if (hit == cache.size()) {
    if (cache.size() >= kGraphCache) {
      cudaGraphExecDestroy(cache.front().exec);
      cache.erase(cache.begin());
    }
    cudaGraph_t graph = nullptr;
    CUDA_TRY(cudaStreamBeginCapture(p->graph_stream, cudaStreamCaptureModeThreadLocal));
    const mgrg_status st = body(p->graph_stream);
    const cudaError_t ce = cudaStreamEndCapture(p->graph_stream, &graph);
    if (st != MGRG_OK) {
      if (graph)
        cudaGraphDestroy(graph);
      return st;
    }
    if (ce != cudaSuccess)
      return fail(MGRG_CUDA_ERROR, std::string("graph capture: ") + cudaGetErrorString(ce));
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess)
      return fail(MGRG_CUDA_ERROR, std::string("graph instantiate: ") + cudaGetErrorString(ie));
    cache.push_back({op, a, b, k, exec, p->last_launches});
    hit = cache.size() - 1;
  } else if (hit + 1 != cache.size()) {
    std::rotate(cache.begin() + hit, cache.begin() + hit + 1, cache.end());
    hit = cache.size() - 1;
  }
  CUDA_TRY(cudaEventRecord(p->graph_ev[0], s));
  CUDA_TRY(cudaStreamWaitEvent(p->graph_stream, p->graph_ev[0], 0));
  CUDA_TRY(cudaGraphLaunch(cache[hit].exec, p->graph_stream));
  CUDA_TRY(cudaEventRecord(p->graph_ev[1], p->graph_stream));
  CUDA_TRY(cudaStreamWaitEvent(s, p->graph_ev[1], 0));
  p->last_launches = cache[hit].launches;
  return MGRG_OK;
}
} // namespace

extern "C" {

mgrg_status mgrg_plan_set_graphs(mgrg_plan *p, int32_t enable) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  DeviceGuard guard(p->device);
  p->graphs = enable != 0;
  if (!p->graphs) {
    for (auto &gr : p->graph_cache)
      cudaGraphExecDestroy(gr.exec);
    p->graph_cache.clear();
  }
  return MGRG_OK;
}

mgrg_status mgrg_decompose(mgrg_plan *p, const void *d_values, void *d_classes,
                           void *stream) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (!d_values || !d_classes)
    return fail(MGRG_INVALID_ARGUMENT, "null device buffer");
  if (p->deferred)
    return fail(p->deferred, p->deferred_msg);
  DeviceGuard guard(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto body = [&](cudaStream_t q) {
    return p->dtype == MGRG_F32
               ? run_decompose<float>(p, static_cast<const float *>(d_values),
                                      static_cast<float *>(d_classes), q)
               : run_decompose<double>(p, static_cast<const double *>(d_values),
                                       static_cast<double *>(d_classes), q);
  };
  if (p->graphs)
    return run_graphed(p, 0, d_values, d_classes, 0, s, body);
  return body(s);
}

mgrg_status mgrg_recompose(mgrg_plan *p, const void *d_classes, int32_t k,
                           void *d_values, void *stream) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (k < 0 || k > p->H.L)
    return fail(MGRG_INVALID_LEVEL, "requested " + std::to_string(k) +
                                        " classes; container has " +
                                        std::to_string(p->H.L));
  if (!d_values || !d_classes)
    return fail(MGRG_INVALID_ARGUMENT, "null device buffer");
  if (p->deferred)
    return fail(p->deferred, p->deferred_msg);
  DeviceGuard guard(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto body = [&](cudaStream_t q) {
    return p->dtype == MGRG_F32
               ? run_recompose<float>(p, static_cast<const float *>(d_classes), k,
                                      static_cast<float *>(d_values), q)
               : run_recompose<double>(p, static_cast<const double *>(d_classes), k,
                                       static_cast<double *>(d_values), q);
  };
  if (p->graphs)
    return run_graphed(p, 1, d_classes, d_values, k, s, body);
  return body(s);
}

// host-API staging: [in | out] with the second half 256-byte aligned (the
// lean finest-level kernels store 2-element vectors)
static uint64_t stage_half(const mgrg_plan *p) {
  return (p->nodes[p->H.L] + 63) & ~uint64_t(63);
}

static mgrg_status ensure_stage(mgrg_plan *p) {
  if (p->d_stage)
    return MGRG_OK;
  const uint64_t n = p->nodes[p->H.L];
  cudaError_t e = cudaMalloc(&p->d_stage, (stage_half(p) + n) * p->esize);
  if (e != cudaSuccess)
    return fail(e == cudaErrorMemoryAllocation ? MGRG_OUT_OF_MEMORY : MGRG_CUDA_ERROR,
                std::string("staging allocation: ") + cudaGetErrorString(e));
  CUDA_TRY(cudaStreamCreateWithFlags(&p->own_stream, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&p->s_in, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking));
  for (int i = 0; i < 16; ++i) {
    CUDA_TRY(cudaEventCreateWithFlags(&p->ev_in[i], cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&p->ev_dec[i], cudaEventDisableTiming));
  }
  CUDA_TRY(cudaEventCreateWithFlags(&p->ev_done, cudaEventDisableTiming));
  p->xfer.reset(new HostXfer(p->device));
  p->xfer->init(p->s_out, n * p->esize);
  return MGRG_OK;
}

extern "C++" {
// Pipelined host-buffer decompose (either policy, dyadic 3-D finest level): the input
// goes up in z slabs on one copy stream, the finest-level kernel runs per
// slab group as soon as its planes (plus one halo plane) are resident, and
// each group's finished class-L pieces (z-major within every class type) go
// down on the other copy stream while later slabs are still uploading --
// PCIe carries both directions at once.  The finest level's Thomas solves
// and the coarser levels follow; classes 0..L-1 (1/8 of the data) last.
// Host buffers are HostViews (hostio.cuh): pinned ones are DMA'd directly,
// pageable ones through the plan's pinned rings; uploads are issued one slab
// ahead of the kernel that needs them, so with pageable memory the host
// copies of later slabs overlap the kernels and downloads of earlier ones.
template <typename R>
mgrg_status decompose_host_pipelined(mgrg_plan *p, const HostView &hin, const HostView &hcls) {
  PlanT<R> &P = pt<R>(p);
  HostXfer &X = *p->xfer;
  const int L = p->H.L;
  const LevelGeom<R> &g = P.geom[L];
  const uint64_t nxy = uint64_t(g.n[0]) * g.n[1];
  R *din = static_cast<R *>(p->d_stage), *dcls = din + stage_half(p);
  R *clsL = dcls + p->nodes[L - 1];
  R *Pout = L == 1 ? dcls : level_buf<R>(p, L - 1);
  R *F = ws<R>(p, p->offF);
  const LeanTiles t = lean_tiles<R>(g.m[0], g.m[1], g.m[2], true);
  // slab groups: 16 measured best on B200 + PCIe 5 (8: 122 ms, 16: 112 ms for
  // 1025^3 f32); MGRG_PIPE_G overrides (1..16, the event arrays' size)
  static const int kG = std::max(1, std::min(16, knob("MGRG_PIPE_G", 16)));
  const int G = int(std::min<uint32_t>(t.ntz, uint32_t(kG)));
  const uint32_t n2 = g.n[2], m2 = g.m[2];
  auto chunk0 = [&](int q) { return uint32_t((uint64_t(q) * t.ntz) / G); };
  auto fplane = [&](uint32_t c) { return std::min<uint32_t>(2 * c * t.zc, n2); };
  cudaStream_t sc = p->own_stream;
  int uploaded = 0;
  auto upload_through = [&](int q) -> mgrg_status {
    for (; uploaded <= q; ++uploaded) {
      const int u = uploaded;
      const uint32_t z0 = fplane(chunk0(u)), z1 = u == G - 1 ? n2 : fplane(chunk0(u + 1));
      CUDA_TRY(X.upload(din + z0 * nxy, hin, z0 * nxy, (z1 - z0) * nxy, p->s_in));
      CUDA_TRY(cudaEventRecord(p->ev_in[u], p->s_in));
    }
    return MGRG_OK;
  };
  for (int q = 0; q < G; ++q) {
    const uint32_t c0 = chunk0(q), c1 = chunk0(q + 1);
    // the group reads fine planes up to 2*c1*zc: the next slab's first plane
    const int need = std::min(q + 1, G - 1);
    if (mgrg_status st = upload_through(need))
      return st;
    CUDA_TRY(cudaStreamWaitEvent(sc, p->ev_in[need], 0));
    LeanTiles tg = t;
    tg.tz0 = c0;
    tg.ntz = c1 - c0;
    const unsigned blocks = unsigned((tg.warps() + kLeanWPB - 1) / kLeanWPB);
    auto k = p->fast ? lean_dec_kernel<R, true, true> : lean_dec_kernel<R, true, false>;
    k<<<blocks, 32 * kLeanWPB, lean_dec_smem<R>(), sc>>>(
        g, P.lean[L][0], P.lean[L][1], P.lean[L][2], P.sten[L][0], P.sten[L][1], P.sten[L][2],
        din, clsL, Pout, F, tg);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(p->ev_dec[q], sc));
    // class-L pieces of coarse z planes [c0*zc, c1*zc): even-z types (1..3)
    // have m2 z ranks, odd-z types (4..7) m2 - 1
    const uint32_t zr0 = c0 * t.zc;
    for (unsigned ty = 1; ty < 8; ++ty) {
      const uint32_t nz = (ty & 4) ? m2 - 1 : m2;
      const uint32_t a = std::min(zr0, nz), b = std::min<uint32_t>(c1 * t.zc, nz);
      if (q == G - 1 && b < nz)
        return fail(MGRG_CUDA_ERROR, "pipelined decompose: slab groups do not cover z");
      if (b <= a)
        continue;
      const uint64_t S = uint64_t(g.tex[ty]) * g.tey[ty];
      const uint64_t off = p->nodes[L - 1] + g.tbase[ty] + S * a;
      CUDA_TRY(X.download(hcls, off, S * (b - a), dcls + off, p->ev_dec[q]));
    }
  }
  // finest level's solves + coarser levels, then classes 0..L-1
  if (mgrg_status st = run_decompose<R>(p, din, dcls, sc, /*top_done=*/true))
    return st;
  CUDA_TRY(cudaEventRecord(p->ev_done, sc));
  CUDA_TRY(X.download(hcls, 0, p->nodes[L - 1], dcls, p->ev_done));
  CUDA_TRY(X.drain());
  CUDA_TRY(cudaStreamSynchronize(sc));
  return MGRG_OK;
}

// Pipelined host-buffer recompose (dyadic 3-D finest level, all classes):
// classes 0..L-1 go up first and the coarse levels run while class L goes up
// in z slab groups; the finest level's load vector is built per group as its
// pieces (plus one halo rank) land, then the solves, then the finest level is
// written per group and each group's output planes go down while later
// groups are still being interpolated.
template <typename R>
mgrg_status recompose_host_pipelined(mgrg_plan *p, const HostView &hcls, const HostView &hout) {
  PlanT<R> &P = pt<R>(p);
  HostXfer &X = *p->xfer;
  const int L = p->H.L;
  const LevelGeom<R> &g = P.geom[L];
  const uint64_t nxy = uint64_t(g.n[0]) * g.n[1];
  R *dcls = static_cast<R *>(p->d_stage), *dout = dcls + stage_half(p);
  R *F = ws<R>(p, p->offF);
  const R *prev = L == 1 ? dcls : level_buf<R>(p, L - 1);
  const R *clsL = dcls + p->nodes[L - 1];
  const uint32_t m2 = g.m[2], n2 = g.n[2];
  cudaStream_t sc = p->own_stream;
  // classes 0..L-1 first; the coarse levels run as soon as they are resident
  CUDA_TRY(X.upload(dcls, hcls, 0, p->nodes[L - 1], p->s_in));
  CUDA_TRY(cudaEventRecord(p->ev_done, p->s_in));
  CUDA_TRY(cudaStreamWaitEvent(sc, p->ev_done, 0));
  if (L > 1)
    if (mgrg_status st = run_recompose<R>(p, dcls, L, dout, sc, L - 1))
      return st;
  // class L by rload chunk groups, each uploaded one group ahead of the
  // finest load-vector kernel that reads it: chunk range [c0, c1) reads class
  // ranks c0-1 .. c1 (the next group's first rank)
  const LeanTiles tr = lean_rtiles<R>(g.m[0], g.m[1], m2, true, p->fast);
  const int G = int(std::min<uint32_t>(tr.ntz, 16));
  auto rchunk0 = [&](int q) { return uint32_t((uint64_t(q) * tr.ntz) / G); };
  int uploaded = 0;
  auto upload_through = [&](int q) -> mgrg_status {
    for (; uploaded <= q; ++uploaded) {
      const int u = uploaded;
      const uint32_t zr0 = rchunk0(u) * tr.zc, zr1 = u == G - 1 ? m2 : rchunk0(u + 1) * tr.zc;
      for (unsigned ty = 1; ty < 8; ++ty) {
        const uint32_t nz = (ty & 4) ? m2 - 1 : m2;
        const uint32_t a = std::min(zr0, nz), b = u == G - 1 ? nz : std::min(zr1, nz);
        if (b <= a)
          continue;
        const uint64_t S = uint64_t(g.tex[ty]) * g.tey[ty];
        const uint64_t off = p->nodes[L - 1] + g.tbase[ty] + S * a;
        CUDA_TRY(X.upload(dcls + off, hcls, off, S * (b - a), p->s_in));
      }
      CUDA_TRY(cudaEventRecord(p->ev_in[u], p->s_in));
    }
    return MGRG_OK;
  };
  for (int q = 0; q < G; ++q) {
    const int need = std::min(q + 1, G - 1);
    if (mgrg_status st = upload_through(need))
      return st;
    CUDA_TRY(cudaStreamWaitEvent(sc, p->ev_in[need], 0));
    LeanTiles t = tr;
    t.tz0 = rchunk0(q);
    t.ntz = rchunk0(q + 1) - rchunk0(q);
    if (q == G - 1)
      t.ntz = tr.ntz - t.tz0;
    const unsigned blocks = unsigned((t.warps() + kLeanWPB - 1) / kLeanWPB);
    auto k = p->fast ? lean_rload_kernel<R, true, true> : lean_rload_kernel<R, true, false>;
    k<<<blocks, 32 * kLeanWPB, 0, sc>>>(g, P.lean[L][0], P.lean[L][1], P.lean[L][2],
                                        P.sten[L][0], P.sten[L][1], P.sten[L][2], clsL, F, t);
    CUDA_TRY(cudaGetLastError());
  }
  for (int i = 0; i < p->nrefine; ++i) {
    const int kd = p->refine_dims[i];
    const bool last = i == p->nrefine - 1;
    launch_thomas<R>(p->fast, g, P.thom[L][kd], P.tlean[L][kd], kd, F,
                     last ? Epi::sub : Epi::none, prev, F, sc, &P.ttp[L][kd]);
  }
  CUDA_TRY(cudaGetLastError());
  // finest level per group, each group's planes [2c0, 2c1) down at once
  const LeanTiles tg = lean_gtiles<R>(g.m[0], g.m[1], m2, true);
  const int H = int(std::min<uint32_t>(tg.ntz, 16));
  auto gchunk0 = [&](int q) { return uint32_t((uint64_t(q) * tg.ntz) / H); };
  for (int q = 0; q < H; ++q) {
    LeanTiles t = tg;
    t.tz0 = gchunk0(q);
    t.ntz = (q == H - 1 ? tg.ntz : gchunk0(q + 1)) - t.tz0;
    const unsigned blocks = unsigned((t.warps() + kLeanWPB - 1) / kLeanWPB);
    auto k = p->fast ? lean_rgpk_kernel<R, true, true, true>
                     : lean_rgpk_kernel<R, true, true, false>;
    k<<<blocks, 32 * kLeanWPB, 0, sc>>>(g, P.lean[L][0], P.lean[L][1], P.lean[L][2], F, clsL,
                                        dout, t);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(p->ev_dec[q], sc));
    const uint32_t z0 = std::min<uint32_t>(2 * t.tz0 * tg.zc, n2);
    const uint32_t z1 = q == H - 1 ? n2 : std::min<uint32_t>(2 * gchunk0(q + 1) * tg.zc, n2);
    if (z1 > z0)
      CUDA_TRY(X.download(hout, z0 * nxy, (z1 - z0) * nxy, dout + z0 * nxy, p->ev_dec[q]));
  }
  CUDA_TRY(X.drain());
  CUDA_TRY(cudaStreamSynchronize(sc));
  return MGRG_OK;
}

template <typename R> bool pipelined_ok(mgrg_plan *p) {
  if (p->gen)
    return false;
  const int L = p->H.L;
  const LevelGeom<R> &g = pt<R>(p).geom[L];
  return p->lean && p->refine == 7u && lean_level(g) && g.n[2] > 1 &&
         p->nodes[L] >= (uint64_t(1) << 22) && g_pipelined_host;
}

// class offsets of the plan's class buffer (class l: [off[l], off[l+1]))
static std::vector<uint64_t> class_offsets(const mgrg_plan *p) {
  std::vector<uint64_t> off(size_t(p->H.L) + 2, 0);
  for (int l = 0; l <= p->H.L; ++l)
    off[size_t(l) + 1] = p->nodes[l];
  return off;
}

static mgrg_status host_views_ok(const HostView &a, const HostView &b) {
  if (a.device || b.device)
    return fail(MGRG_INVALID_ARGUMENT,
                "device pointer passed to a host-buffer entry point (use mgrg_decompose / "
                "mgrg_recompose for device buffers)");
  return MGRG_OK;
}

static mgrg_status host_decompose_impl(mgrg_plan *p, const HostView &hin,
                                       const HostView &hcls) {
  if (mgrg_status st = ensure_stage(p))
    return st;
  if (p->deferred)
    return fail(p->deferred, p->deferred_msg);
  if (p->dtype == MGRG_F32 ? pipelined_ok<float>(p) : pipelined_ok<double>(p))
    return p->dtype == MGRG_F32 ? decompose_host_pipelined<float>(p, hin, hcls)
                                : decompose_host_pipelined<double>(p, hin, hcls);
  HostXfer &X = *p->xfer;
  const uint64_t n = p->nodes[p->H.L];
  char *din = static_cast<char *>(p->d_stage), *dout = din + stage_half(p) * p->esize;
  CUDA_TRY(X.upload(din, hin, 0, n, p->own_stream));
  if (mgrg_status st = mgrg_decompose(p, din, dout, p->own_stream))
    return st;
  CUDA_TRY(cudaEventRecord(p->ev_done, p->own_stream));
  CUDA_TRY(X.download(hcls, 0, n, dout, p->ev_done));
  CUDA_TRY(X.drain());
  CUDA_TRY(cudaStreamSynchronize(p->own_stream));
  return MGRG_OK;
}

static mgrg_status host_recompose_impl(mgrg_plan *p, const HostView &hcls, int32_t k,
                                       const HostView &hout) {
  if (mgrg_status st = ensure_stage(p))
    return st;
  if (k == p->H.L && (p->dtype == MGRG_F32 ? pipelined_ok<float>(p) : pipelined_ok<double>(p)))
    return p->dtype == MGRG_F32 ? recompose_host_pipelined<float>(p, hcls, hout)
                                : recompose_host_pipelined<double>(p, hcls, hout);
  HostXfer &X = *p->xfer;
  char *din = static_cast<char *>(p->d_stage), *dout = din + stage_half(p) * p->esize;
  // only classes 0..k are read (refactor.hpp:483-485): copy that prefix
  CUDA_TRY(X.upload(din, hcls, 0, p->nodes[k], p->own_stream));
  if (mgrg_status st = mgrg_recompose(p, din, k, dout, p->own_stream))
    return st;
  CUDA_TRY(cudaEventRecord(p->ev_done, p->own_stream));
  CUDA_TRY(X.download(hout, 0, p->nodes[p->H.L], dout, p->ev_done));
  CUDA_TRY(X.drain());
  CUDA_TRY(cudaStreamSynchronize(p->own_stream));
  return MGRG_OK;
}
// On failure nothing queued may still touch the caller's buffers after the
// call returns: queued downloads are drained and the copy streams synced
// (their own errors are secondary to the one reported).
static void host_quiesce(mgrg_plan *p) {
  if (p->xfer)
    (void)p->xfer->drain();
  for (cudaStream_t q : {p->s_in, p->s_out, p->own_stream})
    if (q)
      (void)cudaStreamSynchronize(q);
  cudaGetLastError();
}

static mgrg_status host_decompose(mgrg_plan *p, const HostView &hin, const HostView &hcls) {
  if (mgrg_status st = host_views_ok(hin, hcls))
    return st;
  DeviceGuard guard(p->device);
  const mgrg_status st = host_decompose_impl(p, hin, hcls);
  if (st != MGRG_OK) {
    const std::string msg = g_last_error;
    host_quiesce(p);
    g_last_error = msg;
  }
  return st;
}

static mgrg_status host_recompose(mgrg_plan *p, const HostView &hcls, int32_t k,
                                  const HostView &hout) {
  if (mgrg_status st = host_views_ok(hcls, hout))
    return st;
  DeviceGuard guard(p->device);
  const mgrg_status st = host_recompose_impl(p, hcls, k, hout);
  if (st != MGRG_OK) {
    const std::string msg = g_last_error;
    host_quiesce(p);
    g_last_error = msg;
  }
  return st;
}
} // extern "C++"

static mgrg_status check_level_arg(const mgrg_plan *p, int32_t k) {
  if (k < 0 || k > p->H.L)
    return fail(MGRG_INVALID_LEVEL, "requested " + std::to_string(k) +
                                        " classes; container has " +
                                        std::to_string(p->H.L));
  return MGRG_OK;
}

mgrg_status mgrg_decompose_host(mgrg_plan *p, const void *h_values, void *h_classes) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (!h_values || !h_classes)
    return fail(MGRG_INVALID_ARGUMENT, "null host buffer");
  DeviceGuard guard(p->device);
  return host_decompose(p, HostView::of(h_values, p->esize), HostView::of(h_classes, p->esize));
}

mgrg_status mgrg_decompose_host_classes(mgrg_plan *p, const void *h_values,
                                        void *const *h_classes) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (!h_values || !h_classes)
    return fail(MGRG_INVALID_ARGUMENT, "null host buffer");
  const std::vector<uint64_t> off = class_offsets(p);
  for (int l = 0; l <= p->H.L; ++l)
    if (!h_classes[l] && off[size_t(l) + 1] > off[size_t(l)])
      return fail(MGRG_INVALID_ARGUMENT, "null class buffer " + std::to_string(l));
  DeviceGuard guard(p->device);
  return host_decompose(p, HostView::of(h_values, p->esize),
                        HostView::classes(h_classes, off.data(), p->H.L + 1, p->esize));
}

mgrg_status mgrg_recompose_host(mgrg_plan *p, const void *h_classes, int32_t k,
                                void *h_values) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (!h_values || !h_classes)
    return fail(MGRG_INVALID_ARGUMENT, "null host buffer");
  if (mgrg_status st = check_level_arg(p, k))
    return st;
  DeviceGuard guard(p->device);
  return host_recompose(p, HostView::of(h_classes, p->esize), k,
                        HostView::of(h_values, p->esize));
}

mgrg_status mgrg_recompose_host_classes(mgrg_plan *p, const void *const *h_classes, int32_t k,
                                        void *h_values) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (!h_values || !h_classes)
    return fail(MGRG_INVALID_ARGUMENT, "null host buffer");
  if (mgrg_status st = check_level_arg(p, k))
    return st;
  const std::vector<uint64_t> off = class_offsets(p);
  for (int l = 0; l <= k; ++l)
    if (!h_classes[l] && off[size_t(l) + 1] > off[size_t(l)])
      return fail(MGRG_INVALID_ARGUMENT, "null class buffer " + std::to_string(l));
  DeviceGuard guard(p->device);
  return host_recompose(p, HostView::classes(h_classes, off.data(), k + 1, p->esize), k,
                        HostView::of(h_values, p->esize));
}

// ---- split host calls (begin / end) --------------------------------------
// The caller allocates its outputs between the two: _begin uploads the
// inputs (pageable ones through the plan's rings, by the calling thread) and
// enqueues the device path into the plan's staging; _end downloads into the
// caller's buffers and waits.  The drop-in overlaps the reference API's
// output allocation with the upload and the device work this way.
static mgrg_status split_begin_check(mgrg_plan *p) {
  if (p->split_op)
    return fail(MGRG_INVALID_ARGUMENT, "a split host call is already in flight on this plan");
  return MGRG_OK;
}

mgrg_status mgrg_decompose_host_begin(mgrg_plan *p, const void *h_values) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (mgrg_status st = split_begin_check(p))
    return st;
  if (!h_values)
    return fail(MGRG_INVALID_ARGUMENT, "null host buffer");
  const HostView hin = HostView::of(h_values, p->esize);
  if (mgrg_status st = host_views_ok(hin, hin))
    return st;
  DeviceGuard guard(p->device);
  if (mgrg_status st = ensure_stage(p))
    return st;
  if (p->deferred)
    return fail(p->deferred, p->deferred_msg);
  const uint64_t n = p->nodes[p->H.L];
  char *din = static_cast<char *>(p->d_stage), *dout = din + stage_half(p) * p->esize;
  mgrg_status st = MGRG_OK;
  if (cudaError_t e = p->xfer->upload(din, hin, 0, n, p->own_stream))
    st = fail(MGRG_CUDA_ERROR, cudaGetErrorString(e));
  if (!st)
    st = mgrg_decompose(p, din, dout, p->own_stream);
  if (!st)
    if (cudaError_t e = cudaEventRecord(p->ev_done, p->own_stream))
      st = fail(MGRG_CUDA_ERROR, cudaGetErrorString(e));
  if (st) {
    const std::string msg = g_last_error;
    host_quiesce(p);
    g_last_error = msg;
    return st;
  }
  p->split_op = 1;
  return MGRG_OK;
}

mgrg_status mgrg_decompose_host_end(mgrg_plan *p, void *const *h_classes) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (p->split_op != 1)
    return fail(MGRG_INVALID_ARGUMENT, "no mgrg_decompose_host_begin in flight on this plan");
  if (!h_classes)
    return fail(MGRG_INVALID_ARGUMENT, "null host buffer");
  const std::vector<uint64_t> off = class_offsets(p);
  for (int l = 0; l <= p->H.L; ++l)
    if (!h_classes[l] && off[size_t(l) + 1] > off[size_t(l)])
      return fail(MGRG_INVALID_ARGUMENT, "null class buffer " + std::to_string(l));
  const HostView hcls = HostView::classes(h_classes, off.data(), p->H.L + 1, p->esize);
  if (mgrg_status st = host_views_ok(hcls, hcls))
    return st;
  DeviceGuard guard(p->device);
  p->split_op = 0;
  const char *dout = static_cast<const char *>(p->d_stage) + stage_half(p) * p->esize;
  mgrg_status st = MGRG_OK;
  cudaError_t e = p->xfer->download(hcls, 0, p->nodes[p->H.L], dout, p->ev_done);
  if (!e)
    e = p->xfer->drain();
  if (!e)
    e = cudaStreamSynchronize(p->own_stream);
  if (e) {
    st = fail(MGRG_CUDA_ERROR, cudaGetErrorString(e));
    const std::string msg = g_last_error;
    host_quiesce(p);
    g_last_error = msg;
  }
  return st;
}

mgrg_status mgrg_recompose_host_begin(mgrg_plan *p, const void *const *h_classes, int32_t k) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (mgrg_status st = split_begin_check(p))
    return st;
  if (!h_classes)
    return fail(MGRG_INVALID_ARGUMENT, "null host buffer");
  if (mgrg_status st = check_level_arg(p, k))
    return st;
  const std::vector<uint64_t> off = class_offsets(p);
  for (int l = 0; l <= k; ++l)
    if (!h_classes[l] && off[size_t(l) + 1] > off[size_t(l)])
      return fail(MGRG_INVALID_ARGUMENT, "null class buffer " + std::to_string(l));
  const HostView hcls = HostView::classes(h_classes, off.data(), k + 1, p->esize);
  if (mgrg_status st = host_views_ok(hcls, hcls))
    return st;
  DeviceGuard guard(p->device);
  if (mgrg_status st = ensure_stage(p))
    return st;
  char *din = static_cast<char *>(p->d_stage), *dout = din + stage_half(p) * p->esize;
  mgrg_status st = MGRG_OK;
  // only classes 0..k are read (refactor.hpp:483-485)
  if (cudaError_t e = p->xfer->upload(din, hcls, 0, p->nodes[k], p->own_stream))
    st = fail(MGRG_CUDA_ERROR, cudaGetErrorString(e));
  if (!st)
    st = mgrg_recompose(p, din, k, dout, p->own_stream);
  if (!st)
    if (cudaError_t e = cudaEventRecord(p->ev_done, p->own_stream))
      st = fail(MGRG_CUDA_ERROR, cudaGetErrorString(e));
  if (st) {
    const std::string msg = g_last_error;
    host_quiesce(p);
    g_last_error = msg;
    return st;
  }
  p->split_op = 2;
  return MGRG_OK;
}

mgrg_status mgrg_recompose_host_end(mgrg_plan *p, void *h_values) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (p->split_op != 2)
    return fail(MGRG_INVALID_ARGUMENT, "no mgrg_recompose_host_begin in flight on this plan");
  if (!h_values)
    return fail(MGRG_INVALID_ARGUMENT, "null host buffer");
  const HostView hout = HostView::of(h_values, p->esize);
  if (mgrg_status st = host_views_ok(hout, hout))
    return st;
  DeviceGuard guard(p->device);
  p->split_op = 0;
  const char *dout = static_cast<const char *>(p->d_stage) + stage_half(p) * p->esize;
  mgrg_status st = MGRG_OK;
  cudaError_t e = p->xfer->download(hout, 0, p->nodes[p->H.L], dout, p->ev_done);
  if (!e)
    e = p->xfer->drain();
  if (!e)
    e = cudaStreamSynchronize(p->own_stream);
  if (e) {
    st = fail(MGRG_CUDA_ERROR, cudaGetErrorString(e));
    const std::string msg = g_last_error;
    host_quiesce(p);
    g_last_error = msg;
  }
  return st;
}

mgrg_status mgrg_host_abort(mgrg_plan *p) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  DeviceGuard guard(p->device);
  if (p->split_op)
    host_quiesce(p);
  p->split_op = 0;
  return MGRG_OK;
}

// ---- unit-level kernels ------------------------------------------------

static mgrg_status check_level(const mgrg_plan *p, int32_t level) {
  if (level < 1 || level > p->H.L)
    return fail(MGRG_INVALID_LEVEL, "level " + std::to_string(level) + " outside [1, " +
                                        std::to_string(p->H.L) + "]");
  return MGRG_OK;
}

extern "C++" {
template <typename R>
static mgrg_status gpk_t(mgrg_plan *p, int level, int inverse, void *d, cudaStream_t s) {
  if (p->gen) {
    const Gen4Geom<R> &g = pt<R>(p).g4[level];
    gen_gpk_inplace_kernel<R><<<gen_blocks(g.nodes()), 256, 0, s>>>(g, static_cast<R *>(d),
                                                                    inverse);
    CUDA_TRY(cudaGetLastError());
    return MGRG_OK;
  }
  const LevelGeom<R> &g = pt<R>(p).geom[level];
  const uint64_t n = g.nodes();
  gpk_inplace_kernel<R><<<unsigned((n + 255) / 256), 256, 0, s>>>(g, static_cast<R *>(d),
                                                                   inverse);
  CUDA_TRY(cudaGetLastError());
  return MGRG_OK;
}
} // extern "C++"

mgrg_status mgrg_gpk(mgrg_plan *p, int32_t level, int32_t inverse, void *d, void *stream) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (mgrg_status st = check_level(p, level))
    return st;
  if (!d)
    return fail(MGRG_INVALID_ARGUMENT, "null device buffer");
  DeviceGuard guard(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return p->dtype == MGRG_F32 ? gpk_t<float>(p, level, inverse, d, s)
                              : gpk_t<double>(p, level, inverse, d, s);
}

extern "C++" {
template <typename R>
static mgrg_status masstrans_t(mgrg_plan *p, int level, int kd, const void *in, void *out,
                               int fused, void *coef, cudaStream_t s) {
  if (p->gen) {
    // input extents: dims < kd coarse, dims >= kd level-l (kernels.hpp:340-352)
    const Gen4Geom<R> &g = pt<R>(p).g4[level];
    uint32_t e[kGenDims];
    uint64_t ein = 1, eout = 1;
    for (int d = 0; d < kGenDims; ++d) {
      e[d] = d < kd ? g.m[d] : g.n[d];
      ein *= e[d];
      eout *= d == kd ? g.m[d] : e[d];
    }
    const R *src = static_cast<const R *>(in);
    if (!(g.m[kd] < g.n[kd])) { // identity transfer (kernels.hpp:351-354)
      CUDA_TRY(cudaMemcpyAsync(out, src, ein * sizeof(R), cudaMemcpyDeviceToDevice, s));
      return MGRG_OK;
    }
    if (kd == 0) {
      R *W = ws<R>(p, p->offW);
      gen_vecc_kernel<R><<<gen_blocks(g.nodes()), 256, 0, s>>>(
          g, src, W, fused ? static_cast<R *>(coef) : nullptr);
      src = W;
    }
    gen_mass_kernel<R><<<gen_blocks(eout), 256, 0, s>>>(
        g, kd, make_uint4(e[0], e[1], e[2], e[3]), src, static_cast<R *>(out));
    CUDA_TRY(cudaGetLastError());
    return MGRG_OK;
  }
  const LevelGeom<R> &g = pt<R>(p).geom[level];
  uint32_t e[3];
  for (int d = 0; d < 3; ++d)
    e[d] = d < kd ? g.m[d] : g.n[d];
  uint64_t total = 1;
  for (int d = 0; d < 3; ++d)
    total *= d == kd ? g.m[d] : e[d];
  masstrans_kernel<R><<<unsigned((total + 255) / 256), 256, 0, s>>>(
      g, kd, e[0], e[1], e[2], static_cast<const R *>(in), static_cast<R *>(out));
  if (fused && coef) {
    const uint64_t n = g.nodes();
    class_copy_kernel<R><<<unsigned((n + 255) / 256), 256, 0, s>>>(
        g, static_cast<const R *>(in), static_cast<R *>(coef));
  }
  CUDA_TRY(cudaGetLastError());
  return MGRG_OK;
}
} // extern "C++"

mgrg_status mgrg_masstrans(mgrg_plan *p, int32_t level, int32_t dim, const void *d_in,
                           void *d_out, int32_t fused, void *d_coef, void *stream) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (mgrg_status st = check_level(p, level))
    return st;
  if (dim < 0 || dim >= p->H.nd)
    return fail(MGRG_SHAPE_ERROR, "dimension " + std::to_string(dim) + " out of range");
  if (fused && dim != 0)
    return fail(MGRG_INVALID_FUSION, "coefficient copy can only fuse with dimension 0");
  if (!d_in || !d_out)
    return fail(MGRG_INVALID_ARGUMENT, "null device buffer");
  DeviceGuard guard(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return p->dtype == MGRG_F32 ? masstrans_t<float>(p, level, dim, d_in, d_out, fused, d_coef, s)
                              : masstrans_t<double>(p, level, dim, d_in, d_out, fused, d_coef, s);
}

extern "C++" {
template <typename R>
static mgrg_status solve_t(mgrg_plan *p, int level, int kd, void *f, cudaStream_t s) {
  if (p->gen) {
    const Gen4Geom<R> &g = pt<R>(p).g4[level];
    if (!(g.m[kd] < g.n[kd]))
      return MGRG_OK; // identity transfer (kernels.hpp:434-435)
    gen_launch_thomas<R>(g, kd, static_cast<R *>(f), s);
    CUDA_TRY(cudaGetLastError());
    return MGRG_OK;
  }
  const LevelGeom<R> &g = pt<R>(p).geom[level];
  if (!((g.refine >> kd) & 1))
    return MGRG_OK; // identity transfer (kernels.hpp:434-435)
  launch_thomas<R>(p->fast, g, pt<R>(p).thom[level][kd], pt<R>(p).tlean[level][kd], kd,
                   static_cast<R *>(f), Epi::none,
                   nullptr, nullptr, s);
  CUDA_TRY(cudaGetLastError());
  return MGRG_OK;
}
} // extern "C++"

mgrg_status mgrg_solve(mgrg_plan *p, int32_t level, int32_t dim, void *d_f, void *stream) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (mgrg_status st = check_level(p, level))
    return st;
  if (dim < 0 || dim >= p->H.nd)
    return fail(MGRG_SHAPE_ERROR, "dimension " + std::to_string(dim) + " out of range");
  if (!d_f)
    return fail(MGRG_INVALID_ARGUMENT, "null device buffer");
  if (p->deferred)
    return fail(p->deferred, p->deferred_msg);
  DeviceGuard guard(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return p->dtype == MGRG_F32 ? solve_t<float>(p, level, dim, d_f, s)
                              : solve_t<double>(p, level, dim, d_f, s);
}

mgrg_status mgrg_apply_correction(mgrg_plan *p, uint64_t count, void *d_v, const void *d_z,
                                  int32_t sign, void *stream) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (!d_v || !d_z)
    return fail(MGRG_INVALID_ARGUMENT, "null device buffer");
  if (count == 0)
    return MGRG_OK;
  DeviceGuard guard(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const unsigned blocks = unsigned((count + 255) / 256);
  if (p->dtype == MGRG_F32)
    apply_kernel<float><<<blocks, 256, 0, s>>>(count, static_cast<float *>(d_v),
                                               static_cast<const float *>(d_z), sign);
  else
    apply_kernel<double><<<blocks, 256, 0, s>>>(count, static_cast<double *>(d_v),
                                                static_cast<const double *>(d_z), sign);
  CUDA_TRY(cudaGetLastError());
  return MGRG_OK;
}

mgrg_status mgrg_reorder(mgrg_plan *p, int32_t level, int32_t dir, const void *d_in,
                         void *d_out, void *stream) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (mgrg_status st = check_level(p, level))
    return st;
  if (!d_in || !d_out)
    return fail(MGRG_INVALID_ARGUMENT, "null device buffer");
  DeviceGuard guard(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t n = p->nodes[level];
  const unsigned blocks = unsigned((n + 255) / 256);
  if (p->gen) {
    if (p->dtype == MGRG_F32)
      gen_reorder_kernel<float><<<blocks, 256, 0, s>>>(p->pf.g4[level], dir,
                                                       static_cast<const float *>(d_in),
                                                       static_cast<float *>(d_out));
    else
      gen_reorder_kernel<double><<<blocks, 256, 0, s>>>(p->pd.g4[level], dir,
                                                        static_cast<const double *>(d_in),
                                                        static_cast<double *>(d_out));
    CUDA_TRY(cudaGetLastError());
    return MGRG_OK;
  }
  if (p->dtype == MGRG_F32)
    reorder_kernel<float><<<blocks, 256, 0, s>>>(p->pf.geom[level], dir,
                                                 static_cast<const float *>(d_in),
                                                 static_cast<float *>(d_out));
  else
    reorder_kernel<double><<<blocks, 256, 0, s>>>(p->pd.geom[level], dir,
                                                  static_cast<const double *>(d_in),
                                                  static_cast<double *>(d_out));
  CUDA_TRY(cudaGetLastError());
  return MGRG_OK;
}

// ---- cooperative multi-GPU decompose -----------------

} // extern "C"

namespace {

// z solve of one worker's coarse planes for fibers [f0, f1) of the xy plane
// (thomas_fiber, kernels.hpp:143-151, in the reference's order: bit-exact).
// dir 0: v[c] += fwd[c] * v[c-1]; carry_out = v[c1-1].  dir 1: v[m-1] *= ip,
// v[c] = (v[c] - h[c] * v[c+1]) * ip[c], then P[c] += v[c] (apply_pack);
// carry_out = v[c0].
template <typename R>
__global__ void coop_tz_kernel(R *__restrict__ f, R *__restrict__ P, ThomasGeom<R> t,
                               uint64_t m01, uint32_t c0, uint32_t c1, uint64_t f0,
                               uint64_t f1, int dir, const R *__restrict__ cin,
                               R *__restrict__ cout) {
  const uint64_t xy = f0 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (xy >= f1)
    return;
  R *v = f + xy;
  const uint32_t mm = t.m;
  if (dir == 0) {
    R prev = cin ? cin[xy] : R(0);
    for (uint32_t c = c0; c < c1; ++c) {
      R x = v[c * m01];
      if (c > 0)
        x = add(x, mul(t.fwd[c], prev));
      v[c * m01] = x;
      prev = x;
    }
    if (cout)
      cout[xy] = prev;
  } else {
    R next = cin ? cin[xy] : R(0);
    for (uint32_t c = c1; c-- > c0;) {
      R x = v[c * m01];
      x = c == mm - 1 ? mul(x, t.ip[c]) : mul(sub(x, mul(t.h[c], next)), t.ip[c]);
      v[c * m01] = x;
      P[xy + c * m01] = add(P[xy + c * m01], x);
      next = x;
    }
    if (cout)
      cout[xy] = next;
  }
}

template <typename R>
mgrg_status coop_level_t(mgrg_plan *p, int l, uint32_t c0, uint32_t c1, const R *d_level,
                         R *d_cls, cudaStream_t s) {
  PlanT<R> &P = pt<R>(p);
  const int L = p->H.L;
  const LevelGeom<R> &g = P.geom[l];
  if (!(p->lean && p->refine == 7u && lean_level(g)))
    return fail(MGRG_UNSUPPORTED, "cooperative levels need a 3-D grid with odd extents "
                                  "refining in every dimension");
  const uint32_t m2 = g.m[2];
  if (!(c0 < c1 && c1 <= m2))
    return fail(MGRG_INVALID_ARGUMENT, "coarse plane range out of bounds");
  const R *a = l == L ? d_level : level_buf<R>(p, l);
  if (!a)
    return fail(MGRG_INVALID_ARGUMENT, "null level array");
  if ((reinterpret_cast<uintptr_t>(a) & 15) != 0)
    return fail(MGRG_INVALID_ARGUMENT, "level array must be 16-byte aligned");
  R *Pout = l == 1 ? d_cls : level_buf<R>(p, l - 1);
  R *F = ws<R>(p, p->offF);
  R *cls = d_cls + p->nodes[l - 1];
  LeanTiles t = lean_tiles<R>(g.m[0], g.m[1], g.m[2], true);
  uint32_t zc = t.zc;
  while (zc > 1 && (c0 % zc || (c1 < m2 && c1 % zc)))
    zc >>= 1;
  t.zc = zc;
  t.tz0 = c0 / zc;
  t.ntz = (c1 - c0 + zc - 1) / zc;
  const unsigned blocks = unsigned((t.warps() + kLeanWPB - 1) / kLeanWPB);
  if (p->fast)
    lean_dec_kernel<R, true, true><<<blocks, 32 * kLeanWPB, lean_dec_smem<R>(), s>>>(
        g, P.lean[l][0], P.lean[l][1], P.lean[l][2], P.sten[l][0], P.sten[l][1], P.sten[l][2],
        a, cls, Pout, F, t);
  else
    lean_dec_kernel<R, true, false><<<blocks, 32 * kLeanWPB, lean_dec_smem<R>(), s>>>(
        g, P.lean[l][0], P.lean[l][1], P.lean[l][2], P.sten[l][0], P.sten[l][1], P.sten[l][2],
        a, cls, Pout, F, t);
  CUDA_TRY(cudaGetLastError());
  // x and y solves of the worker's planes: the exact-order kernels on the
  // sub-lattice (the FAST chunked kernels assume a 16-byte aligned lattice)
  LevelGeom<R> gs = g;
  gs.m[2] = c1 - c0;
  R *Fs = F + uint64_t(c0) * g.m[0] * g.m[1];
  for (int kd = 0; kd < 2; ++kd)
    launch_thomas<R>(false, gs, P.thom[l][kd], P.tlean[l][kd], kd, Fs, Epi::none, nullptr,
                     nullptr, s);
  CUDA_TRY(cudaGetLastError());
  return MGRG_OK;
}

template <typename R>
mgrg_status coop_tz_t(mgrg_plan *p, int l, uint32_t c0, uint32_t c1, uint64_t f0, uint64_t f1,
                      int dir, const R *cin, R *cout, R *d_cls, cudaStream_t s) {
  PlanT<R> &P = pt<R>(p);
  const LevelGeom<R> &g = P.geom[l];
  const uint64_t m01 = uint64_t(g.m[0]) * g.m[1];
  if (!(c0 < c1 && c1 <= g.m[2]) || f1 > m01 || f0 >= f1)
    return fail(MGRG_INVALID_ARGUMENT, "plane or fiber range out of bounds");
  R *Pout = l == 1 ? d_cls : level_buf<R>(p, l - 1);
  R *F = ws<R>(p, p->offF);
  coop_tz_kernel<R><<<unsigned((f1 - f0 + 255) / 256), 256, 0, s>>>(
      F, Pout, P.thom[l][2], m01, c0, c1, f0, f1, dir, cin, cout);
  CUDA_TRY(cudaGetLastError());
  return MGRG_OK;
}

} // namespace

extern "C" {

mgrg_status mgrg_coop_level(mgrg_plan *p, int32_t level, uint32_t c0, uint32_t c1,
                            const void *d_level, void *d_classes, void *stream) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (mgrg_status st = check_level(p, level))
    return st;
  if (!d_classes)
    return fail(MGRG_INVALID_ARGUMENT, "null device buffer");
  if (p->deferred)
    return fail(p->deferred, p->deferred_msg);
  if (p->gen)
    return fail(MGRG_UNSUPPORTED, "cooperative decompose of 4-D grids");
  DeviceGuard guard(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return p->dtype == MGRG_F32
             ? coop_level_t<float>(p, level, c0, c1, static_cast<const float *>(d_level),
                                   static_cast<float *>(d_classes), s)
             : coop_level_t<double>(p, level, c0, c1, static_cast<const double *>(d_level),
                                    static_cast<double *>(d_classes), s);
}

mgrg_status mgrg_coop_thomas_z(mgrg_plan *p, int32_t level, uint32_t c0, uint32_t c1,
                               uint64_t f0, uint64_t f1, int32_t direction,
                               const void *d_carry_in, void *d_carry_out, void *d_classes,
                               void *stream) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (mgrg_status st = check_level(p, level))
    return st;
  if (!d_classes)
    return fail(MGRG_INVALID_ARGUMENT, "null device buffer");
  if (p->gen)
    return fail(MGRG_UNSUPPORTED, "cooperative decompose of 4-D grids");
  DeviceGuard guard(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return p->dtype == MGRG_F32
             ? coop_tz_t<float>(p, level, c0, c1, f0, f1, direction,
                                static_cast<const float *>(d_carry_in),
                                static_cast<float *>(d_carry_out),
                                static_cast<float *>(d_classes), s)
             : coop_tz_t<double>(p, level, c0, c1, f0, f1, direction,
                                 static_cast<const double *>(d_carry_in),
                                 static_cast<double *>(d_carry_out),
                                 static_cast<double *>(d_classes), s);
}

mgrg_status mgrg_plan_level_buffer(mgrg_plan *p, int32_t level, void **d_ptr) {
  if (mgrg_status st = check_plan(p))
    return st;
  if (level < 1 || level >= p->H.L || !d_ptr)
    return fail(MGRG_INVALID_ARGUMENT, "level buffer index outside [1, L)");
  *d_ptr = p->dtype == MGRG_F32 ? static_cast<void *>(level_buf<float>(p, level))
                                : static_cast<void *>(level_buf<double>(p, level));
  return MGRG_OK;
}

} // extern "C"

#include "coop_host.cuh"
#include "container.cuh"
#include "compress.cuh"
#include "comm.cuh"
