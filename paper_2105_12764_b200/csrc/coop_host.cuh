// coop_host.cuh -- native cooperative decompose:
// mgrg_cooperative_decompose_host, the C-ABI runtime behind
// mgr::cooperative_decompose in include/mgr_b200/parallel.hpp.
//
// Same algorithm as paper_2105_12764_b200/coop.py (one host thread drives W
// workers, worker w on device (desc.device + w) mod the visible devices):
// z slabs on multiples of 2^q finest planes; per cooperative level the
// 2 + 1 halo planes move between neighbours (cudaMemcpyPeer: NVLink between
// GPUs, a device copy on one GPU), mgrg_coop_level runs on every worker, the
// z solve is chained up (forward elimination) and down (back substitution +
// apply) with one xy carry plane per hop; then the level-(L-q) lattice and
// the class fragments are gathered on worker 0, which finishes the coarse
// levels with a plan for that lattice.  Bit-identical to mgrg_decompose of
// the whole grid (exact policy).  Included at the end of mgrg.cu.
#pragma once

#include <functional>

namespace {

struct CoopGeo {
  int L = 0, q = 0, W = 1;
  std::vector<std::array<uint64_t, 3>> ls; // level shapes
  std::vector<uint64_t> bounds;            // finest-plane slab boundaries
  // coarse planes of worker r at cooperative level L - j
  std::pair<uint64_t, uint64_t> range(int r, int j) const {
    const uint64_t m2 = ls[L - j - 1][2];
    const uint64_t c0 = bounds[r] >> (j + 1);
    const uint64_t c1 = r == W - 1 ? m2 : bounds[r + 1] >> (j + 1);
    return {c0, c1};
  }
};

// coop_levels / slab_bounds of coop.py
int coop_depth(const std::vector<std::array<uint64_t, 3>> &ls, int W) {
  const int L = int(ls.size()) - 1;
  const uint64_t n2 = ls[L][2];
  if (n2 < 3)
    return 0;
  int q = 0;
  while (q < L) {
    const int nq = q + 1;
    if ((n2 - 1) % (uint64_t(1) << nq) || ((n2 - 1) >> nq) < uint64_t(W))
      break;
    const auto &a = ls[L - q], &c = ls[L - q - 1];
    bool ok = true;
    for (int d = 0; d < 3; ++d)
      ok = ok && (a[d] % 2 == 1) && c[d] < a[d];
    if (!ok)
      break;
    q = nq;
  }
  return q;
}

// class-l fragments written by the worker owning coarse planes [c0, c1)
void coop_pieces(const std::array<uint64_t, 3> &ls, uint64_t c0, uint64_t c1, uint64_t m2,
                 std::vector<std::pair<uint64_t, uint64_t>> &out) {
  uint64_t off = 0;
  for (unsigned mask = 1; mask < 8; ++mask) {
    uint64_t e[3];
    for (int d = 0; d < 3; ++d) {
      const uint64_t n = ls[d], ce = n / 2 + 1;
      e[d] = ((mask >> d) & 1) ? n - ce : ce;
    }
    const uint64_t S = e[0] * e[1];
    uint64_t a = c0, b = c1;
    if (mask & 4) {
      a = std::min(c0, m2 - 1);
      b = std::min(c1, m2 - 1);
    }
    if (b > a && S)
      out.push_back({off + S * a, S * (b - a)});
    off += e[0] * e[1] * e[2];
  }
}

struct CoopWorker {
  mgrg_plan *p = nullptr;
  int dev = 0;
  char *in = nullptr, *cls = nullptr, *carry = nullptr; // carry: [in | out] planes
};

} // namespace

extern "C" {

mgrg_status mgrg_cooperative_decompose_host(const mgrg_grid_desc *desc, int32_t workers,
                                            const void *h_values, void *h_classes,
                                            mgrg_fault_fn fault, void *fault_ctx,
                                            uint64_t *remote_elements) {
  g_last_error.clear();
  if (!desc || !h_values || !h_classes)
    return fail(MGRG_INVALID_ARGUMENT, "null argument");
  if (workers < 1)
    return fail(MGRG_TOO_MANY_WORKERS, "worker count must be positive");
  if (desc->ndims >= 1 && desc->ndims <= 4 && workers > 1 &&
      uint64_t(workers) > desc->shape[desc->ndims - 1])
    return fail(MGRG_TOO_MANY_WORKERS,
                "cannot split dimension " + std::to_string(desc->ndims - 1) + " of extent " +
                    std::to_string(desc->shape[desc->ndims - 1]) + " across " +
                    std::to_string(workers) + " workers");
  int ndev = 1;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  const int W = workers;
  std::vector<CoopWorker> wk(W);
  mgrg_plan *sub = nullptr;
  uint64_t moved = 0;
  auto cleanup = [&]() {
    for (auto &w : wk) {
      DeviceGuard g(w.dev);
      cudaFree(w.in);
      cudaFree(w.cls);
      cudaFree(w.carry);
      mgrg_plan_destroy(w.p);
    }
    mgrg_plan_destroy(sub);
  };
  auto phase = [&](int w, const char *name, int level) -> mgrg_status {
    if (fault && fault(fault_ctx, w, name, level) != 0)
      return fail(MGRG_WORKER_FAILURE, "worker " + std::to_string(w) + " failed in " + name);
    return MGRG_OK;
  };
  mgrg_status st = MGRG_OK;
#define COOP_TRY(expr)                                                          \
  do {                                                                         \
    if ((st = (expr)) != MGRG_OK) {                                            \
      const std::string m = g_last_error;                                      \
      cleanup();                                                               \
      g_last_error = m;                                                        \
      return st;                                                               \
    }                                                                          \
  } while (0)
#define COOP_CUDA(expr)                                                        \
  do {                                                                         \
    cudaError_t e_ = (expr);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      cleanup();                                                               \
      return fail(e_ == cudaErrorMemoryAllocation ? MGRG_OUT_OF_MEMORY : MGRG_CUDA_ERROR, \
                  std::string(#expr) + ": " + cudaGetErrorString(e_));         \
    }                                                                          \
  } while (0)
  for (int w = 0; w < W; ++w) {
    mgrg_grid_desc d = *desc;
    d.device = (desc->device + w) % ndev;
    wk[w].dev = d.device;
    COOP_TRY(mgrg_plan_create(&d, &wk[w].p));
  }
  mgrg_plan *p0 = wk[0].p;
  const int L = p0->H.L;
  const uint64_t es = uint64_t(p0->esize), N = p0->nodes[L];
  CoopGeo G;
  G.L = L;
  G.W = W;
  if (p0->H.nd == 3)
    for (int l = 0; l <= L; ++l)
      G.ls.push_back({p0->H.ext[l][0], p0->H.ext[l][1], p0->H.ext[l][2]});
  G.q = (W > 1 && p0->H.nd == 3 && !p0->gen && p0->lean) ? coop_depth(G.ls, W) : 0;
  if (G.q == 0) { // nothing to split on coarse planes: worker 0 alone
    COOP_TRY(phase(0, "serial", L));
    COOP_TRY(mgrg_decompose_host(p0, h_values, h_classes));
    cleanup();
    if (remote_elements)
      *remote_elements = 0;
    return MGRG_OK;
  }
  const int q = G.q;
  {
    const uint64_t n2 = G.ls[L][2], units = (n2 - 1) >> q;
    for (int r = 0; r < W; ++r)
      G.bounds.push_back(((units / W) * r + std::min<uint64_t>(r, units % W)) << q);
    G.bounds.push_back(n2 - 1);
  }
  const uint64_t m01L = G.ls[L - 1][0] * G.ls[L - 1][1];
  for (auto &w : wk) {
    DeviceGuard g(w.dev);
    COOP_CUDA(cudaMalloc(&w.in, N * es));
    COOP_CUDA(cudaMalloc(&w.cls, N * es));
    COOP_CUDA(cudaMalloc(&w.carry, 2 * m01L * es));
  }
  auto copy = [&](int dst, char *dp, int src, const char *sp, uint64_t bytes) -> cudaError_t {
    if (dst != src)
      moved += bytes / es;
    return cudaMemcpyPeer(dp, wk[dst].dev, sp, wk[src].dev, bytes);
  };
  auto level_arr = [&](int w, int l) -> char * {
    if (l == L)
      return wk[w].in;
    if (l == 0)
      return wk[w].cls;
    void *ptr = nullptr;
    mgrg_plan_level_buffer(wk[w].p, l, &ptr);
    return static_cast<char *>(ptr);
  };
  // Define every byte the level kernels may stage: their 16-byte row chunks
  // straddle the first / last plane a worker holds, so the neighbouring
  // (never used) bytes must not be uninitialised memory (compute-sanitizer
  // initcheck).  One HBM-speed pass per worker buffer.
  for (int w = 0; w < W; ++w) {
    DeviceGuard g(wk[w].dev);
    COOP_CUDA(cudaMemset(wk[w].in, 0, N * es));
    for (int l = L - 1; l >= std::max(1, L - 2); --l)
      COOP_CUDA(cudaMemset(level_arr(w, l), 0,
                           G.ls[l][0] * G.ls[l][1] * G.ls[l][2] * es));
  }
  // upload: fine planes [2c0 - 2, 2c1] of the finest level
  {
    const uint64_t nxy = G.ls[L][0] * G.ls[L][1], n2 = G.ls[L][2];
    for (int r = 0; r < W; ++r) {
      const auto [c0, c1] = G.range(r, 0);
      const uint64_t a = c0 ? 2 * c0 - 2 : 0, b = std::min(2 * c1 + 1, n2);
      DeviceGuard g(wk[r].dev);
      COOP_CUDA(cudaMemcpy(wk[r].in + a * nxy * es,
                           static_cast<const char *>(h_values) + a * nxy * es,
                           (b - a) * nxy * es, cudaMemcpyHostToDevice));
    }
  }
  for (int j = 0; j < q; ++j) {
    const int l = L - j;
    const uint64_t lxy = G.ls[l][0] * G.ls[l][1];
    const uint64_t m01 = G.ls[l - 1][0] * G.ls[l - 1][1];
    if (j > 0) // halo planes of the level-l array
      for (int r = 1; r < W; ++r) {
        const uint64_t c0 = G.range(r, j).first;
        COOP_CUDA(copy(r, level_arr(r, l) + (2 * c0 - 2) * lxy * es, r - 1,
                       level_arr(r - 1, l) + (2 * c0 - 2) * lxy * es, 2 * lxy * es));
        COOP_CUDA(copy(r - 1, level_arr(r - 1, l) + 2 * c0 * lxy * es, r,
                       level_arr(r, l) + 2 * c0 * lxy * es, lxy * es));
      }
    for (int r = 0; r < W; ++r) {
      COOP_TRY(phase(r, "level", l));
      const auto [c0, c1] = G.range(r, j);
      COOP_TRY(mgrg_coop_level(wk[r].p, l, uint32_t(c0), uint32_t(c1),
                               l == L ? wk[r].in : nullptr, wk[r].cls, nullptr));
    }
    for (int dir = 0; dir < 2; ++dir)
      for (int k = 0; k < W; ++k) {
        const int r = dir == 0 ? k : W - 1 - k, prev = dir == 0 ? r - 1 : r + 1;
        const bool has_prev = prev >= 0 && prev < W;
        COOP_TRY(phase(r, "solve", l));
        if (has_prev)
          COOP_CUDA(copy(r, wk[r].carry, prev, wk[prev].carry + m01L * es, m01 * es));
        const auto [c0, c1] = G.range(r, j);
        COOP_TRY(mgrg_coop_thomas_z(wk[r].p, l, uint32_t(c0), uint32_t(c1), 0, m01, dir,
                                    has_prev ? wk[r].carry : nullptr,
                                    wk[r].carry + m01L * es, wk[r].cls, nullptr));
      }
    for (auto &w : wk) {
      DeviceGuard g(w.dev);
      COOP_CUDA(cudaDeviceSynchronize());
    }
  }
  // the level-(L-q) lattice on worker 0, then its own decompose
  const int lq = L - q;
  {
    const uint64_t lxy = G.ls[lq][0] * G.ls[lq][1];
    for (int r = 1; r < W; ++r) {
      const auto [c0, c1] = G.range(r, q - 1);
      COOP_CUDA(copy(0, level_arr(0, lq) + c0 * lxy * es, r, level_arr(r, lq) + c0 * lxy * es,
                     (c1 - c0) * lxy * es));
    }
  }
  if (lq >= 1) {
    COOP_TRY(phase(0, "tail", lq));
    std::vector<double> coords;
    for (int d = 0; d < 3; ++d) {
      std::vector<uint64_t> idx(p0->H.shape[d]);
      for (uint64_t i = 0; i < idx.size(); ++i)
        idx[i] = i;
      for (int s = 0; s < q; ++s) {
        std::vector<uint64_t> nx;
        for (size_t i = 0; i < idx.size(); i += 2)
          nx.push_back(idx[i]);
        if (nx.back() != idx.back())
          nx.push_back(idx.back());
        idx.swap(nx);
      }
      for (uint64_t i : idx)
        coords.push_back(p0->H.coords[d][i]);
    }
    mgrg_grid_desc d = *desc;
    d.device = wk[0].dev;
    for (int k = 0; k < 3; ++k)
      d.shape[k] = G.ls[lq][k];
    d.coords = coords.data();
    d.levels = lq;
    COOP_TRY(mgrg_plan_create(&d, &sub));
    if (sub->H.L != lq)
      COOP_TRY(fail(MGRG_INVALID_LEVEL, "coarse tail hierarchy depth mismatch"));
    DeviceGuard g(wk[0].dev);
    COOP_TRY(mgrg_decompose(sub, level_arr(0, lq), wk[0].cls, nullptr));
  }
  // class fragments of the cooperative levels
  for (int j = 0; j < q; ++j) {
    const int l = L - j;
    const uint64_t m2 = G.ls[l - 1][2], base = p0->nodes[l - 1];
    for (int r = 1; r < W; ++r) {
      std::vector<std::pair<uint64_t, uint64_t>> pcs;
      const auto [c0, c1] = G.range(r, j);
      coop_pieces(G.ls[l], c0, c1, m2, pcs);
      for (const auto &[o, n] : pcs)
        COOP_CUDA(copy(0, wk[0].cls + (base + o) * es, r, wk[r].cls + (base + o) * es, n * es));
    }
  }
  {
    DeviceGuard g(wk[0].dev);
    COOP_CUDA(cudaMemcpy(h_classes, wk[0].cls, N * es, cudaMemcpyDeviceToHost));
  }
#undef COOP_TRY
#undef COOP_CUDA
  cleanup();
  if (remote_elements)
    *remote_elements = moved;
  return MGRG_OK;
}

} // extern "C"
