// ref_harness.cpp -- C ABI around the UNMODIFIED reference implementation
// (TEST INFRASTRUCTURE).  Compiled by oracle/Makefile together with
// /root/reference/proj/src/grid.cpp and refactor.cpp (read in place, never
// copied) into oracle/_ref/libmgr_ref.so, with the reference's own flags
// (-std=gnu++20 -O3 -DNDEBUG, no -march: no FMA contraction).  Used to pin
// the C restatement (mgr_oracle.c) and as bench.py's reference arm.
//
// Same argument conventions and status codes as mgr_oracle.h.
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <thread>
#include <vector>

#include "mgr/parallel.hpp"
#include "mgr/pipeline.hpp"
#include "mgr/refactor.hpp"
#include "oracle.hpp" // reference tests/oracle.hpp: deterministic data helpers

namespace {

int code_of(const mgr::Error &e) {
  static const char *names[] = {"",           "InvalidGrid",   "InvalidLevel",
                                "ShapeError", "InvalidFusion", "SingularSystem",
                                "TooManyWorkers", "WorkerFailure", "CorruptFile",
                                "MissingClass", "InvalidBound",  "IoError"};
  for (int i = 1; i < 12; ++i)
    if (e.code() == names[i])
      return i;
  return 15;
}

mgr::Shape to_shape(int nd, const uint64_t *shape) {
  return mgr::Shape(shape, shape + nd);
}

std::vector<std::vector<double>> to_coords(int nd, const uint64_t *shape,
                                           const double *coords) {
  std::vector<std::vector<double>> c;
  for (int d = 0; d < nd; ++d) {
    if (coords) {
      c.emplace_back(coords, coords + shape[d]);
      coords += shape[d];
    } else {
      c.push_back(mgr::uniform_coords(shape[d]));
    }
  }
  return c;
}

template <typename Real>
int decompose_impl(int nd, const uint64_t *shape, const double *coords,
                   int levels_cap, const Real *values, Real *classes,
                   int *levels_out) {
  try {
    mgr::TensorGrid<Real> g;
    g.shape = to_shape(nd, shape);
    g.coords = to_coords(nd, shape, coords);
    g.values.assign(values, values + mgr::num_elements(g.shape));
    mgr::RefactorOptions opt;
    if (levels_cap > 0)
      opt.levels = std::size_t(levels_cap);
    const auto r = mgr::decompose(g, opt);
    std::size_t off = 0;
    for (const auto &c : r.classes) {
      std::memcpy(classes + off, c.data(), c.size() * sizeof(Real));
      off += c.size();
    }
    if (levels_out)
      *levels_out = int(r.levels);
    return 0;
  } catch (const mgr::Error &e) {
    return code_of(e);
  } catch (...) {
    return 15;
  }
}

// decompose_spatiotemporal (refactor.hpp:536-567): nsnap snapshots of one
// nd-D grid, values snapshot-major
template <typename Real>
int spatiotemporal_impl(int nd, const uint64_t *shape, const double *coords, int nsnap,
                        const double *time_coords, const Real *values, Real *classes,
                        int *levels_out) {
  try {
    std::vector<mgr::TensorGrid<Real>> snaps(nsnap);
    const std::size_t n = mgr::num_elements(to_shape(nd, shape));
    for (int t = 0; t < nsnap; ++t) {
      snaps[t].shape = to_shape(nd, shape);
      snaps[t].coords = to_coords(nd, shape, coords);
      snaps[t].values.assign(values + t * n, values + (t + 1) * n);
    }
    const std::vector<double> tc(time_coords, time_coords + nsnap);
    const auto r = mgr::decompose_spatiotemporal(snaps, tc);
    std::size_t off = 0;
    for (const auto &c : r.classes) {
      std::memcpy(classes + off, c.data(), c.size() * sizeof(Real));
      off += c.size();
    }
    if (levels_out)
      *levels_out = int(r.levels);
    return 0;
  } catch (const mgr::Error &e) {
    return code_of(e);
  } catch (...) {
    return 15;
  }
}

template <typename Real>
int recompose_impl(int nd, const uint64_t *shape, const double *coords,
                   int levels, const Real *classes, int k, Real *values) {
  try {
    mgr::RefactoredData<Real> r;
    r.shape = to_shape(nd, shape);
    r.coords = to_coords(nd, shape, coords);
    r.levels = std::size_t(levels);
    const auto hier = mgr::build_hierarchy(r.shape, r.coords,
                                           std::optional<std::size_t>(levels), 2);
    std::size_t off = 0;
    for (std::size_t l = 0; l <= r.levels; ++l) {
      const std::size_t sz =
          l == 0 ? hier.num_nodes(0) : hier.num_nodes(l) - hier.num_nodes(l - 1);
      r.classes.emplace_back(classes + off, classes + off + sz);
      off += sz;
    }
    if (k < 0)
      return 2;
    const auto g = mgr::recompose(r, std::size_t(k));
    std::memcpy(values, g.values.data(), g.values.size() * sizeof(Real));
    return 0;
  } catch (const mgr::Error &e) {
    return code_of(e);
  } catch (...) {
    return 15;
  }
}

template <typename Real>
int gpk_impl(int nd, const uint64_t *shape, const double *coords, int cap,
             int level, int inverse, Real *values) {
  try {
    std::optional<std::size_t> lv;
    if (cap > 0)
      lv = std::size_t(cap);
    const auto hier =
        mgr::build_hierarchy(to_shape(nd, shape), to_coords(nd, shape, coords), lv);
    const std::size_t n = hier.num_nodes(std::size_t(level));
    std::span<Real> s(values, n);
    if (inverse)
      mgr::restore_coefficients<Real>(s, hier, std::size_t(level));
    else
      mgr::compute_coefficients<Real>(s, hier, std::size_t(level));
    return 0;
  } catch (const mgr::Error &e) {
    return code_of(e);
  } catch (...) {
    return 15;
  }
}

template <typename Real>
int masstrans_impl(int nd, const uint64_t *shape, const double *coords, int cap,
                   int level, int dim, const Real *in, Real *out, int fused,
                   Real *coef) {
  try {
    std::optional<std::size_t> lv;
    if (cap > 0)
      lv = std::size_t(cap);
    const auto hier =
        mgr::build_hierarchy(to_shape(nd, shape), to_coords(nd, shape, coords), lv);
    mgr::NdBuffer<Real> b(mgr::masstrans_input_shape(hier, std::size_t(level),
                                                     std::size_t(dim)));
    b.data.assign(in, in + b.data.size());
    std::vector<Real> cv;
    const auto o = mgr::masstrans_apply(b, hier, std::size_t(level),
                                        std::size_t(dim), fused != 0,
                                        coef ? &cv : nullptr);
    std::memcpy(out, o.data.data(), o.data.size() * sizeof(Real));
    if (coef && fused)
      std::memcpy(coef, cv.data(), cv.size() * sizeof(Real));
    return 0;
  } catch (const mgr::Error &e) {
    return code_of(e);
  } catch (...) {
    return 15;
  }
}

template <typename Real>
int solve_impl(int nd, const uint64_t *shape, const double *coords, int cap,
               int level, int dim, Real *f) {
  try {
    std::optional<std::size_t> lv;
    if (cap > 0)
      lv = std::size_t(cap);
    const auto hier =
        mgr::build_hierarchy(to_shape(nd, shape), to_coords(nd, shape, coords), lv);
    mgr::NdBuffer<Real> b(hier.level_shape(std::size_t(level) - 1));
    b.data.assign(f, f + b.data.size());
    mgr::solve_correction(b, hier, std::size_t(level), std::size_t(dim));
    std::memcpy(f, b.data.data(), b.data.size() * sizeof(Real));
    return 0;
  } catch (const mgr::Error &e) {
    return code_of(e);
  } catch (...) {
    return 15;
  }
}

} // namespace

namespace {
// MGRF container (pipeline.cpp:180-300): write the RefactoredData given by
// its flat class buffer (class l at N_{l-1}) with the reference writer.
template <typename Real>
int64_t write_impl(int nd, const uint64_t *shape, const double *coords, int levels,
                   const Real *classes, const char *path) {
  try {
    mgr::RefactoredData<Real> r;
    r.shape = to_shape(nd, shape);
    r.coords = to_coords(nd, shape, coords);
    r.levels = std::size_t(levels);
    const auto hier = mgr::build_hierarchy(r.shape, r.coords,
                                           std::optional<std::size_t>(levels), 2);
    std::size_t off = 0;
    for (std::size_t l = 0; l <= r.levels; ++l) {
      const std::size_t sz =
          l == 0 ? hier.num_nodes(0) : hier.num_nodes(l) - hier.num_nodes(l - 1);
      r.classes.emplace_back(classes + off, classes + off + sz);
      off += sz;
    }
    return int64_t(mgr::write_refactored(r, path));
  } catch (const mgr::Error &e) {
    return -int64_t(code_of(e));
  } catch (...) {
    return -15;
  }
}

// compress / decompress (pipeline.hpp:149-198, pipeline.cpp:517-547)
template <typename Real>
int64_t compress_impl(int nd, const uint64_t *shape, const double *coords, const Real *values,
                      double eb, int codec, uint8_t *out, uint64_t cap, double *bin,
                      double *measured) {
  try {
    mgr::TensorGrid<Real> g;
    g.shape = to_shape(nd, shape);
    g.coords = to_coords(nd, shape, coords);
    g.values.assign(values, values + mgr::num_elements(g.shape));
    const auto r = mgr::compress(g, eb, mgr::codec_by_id(uint8_t(codec)));
    if (r.bytes.size() > cap)
      return -16;
    std::memcpy(out, r.bytes.data(), r.bytes.size());
    *bin = r.report.bin_width;
    *measured = r.report.measured_max_abs_error;
    return int64_t(r.bytes.size());
  } catch (const mgr::Error &e) {
    return -int64_t(code_of(e));
  } catch (...) {
    return -15;
  }
}
} // namespace

extern "C" {

int mgrref_decompose_f64(int nd, const uint64_t *shape, const double *coords,
                         int cap, const double *v, double *c, int *lo) {
  return decompose_impl<double>(nd, shape, coords, cap, v, c, lo);
}
int mgrref_decompose_f32(int nd, const uint64_t *shape, const double *coords,
                         int cap, const float *v, float *c, int *lo) {
  return decompose_impl<float>(nd, shape, coords, cap, v, c, lo);
}
int mgrref_spatiotemporal_f64(int nd, const uint64_t *shape, const double *coords, int nsnap,
                              const double *tc, const double *v, double *c, int *lo) {
  return spatiotemporal_impl<double>(nd, shape, coords, nsnap, tc, v, c, lo);
}
int mgrref_spatiotemporal_f32(int nd, const uint64_t *shape, const double *coords, int nsnap,
                              const double *tc, const float *v, float *c, int *lo) {
  return spatiotemporal_impl<float>(nd, shape, coords, nsnap, tc, v, c, lo);
}
int mgrref_recompose_f64(int nd, const uint64_t *shape, const double *coords,
                         int levels, const double *c, int k, double *v) {
  return recompose_impl<double>(nd, shape, coords, levels, c, k, v);
}
int mgrref_recompose_f32(int nd, const uint64_t *shape, const double *coords,
                         int levels, const float *c, int k, float *v) {
  return recompose_impl<float>(nd, shape, coords, levels, c, k, v);
}
int mgrref_gpk_f64(int nd, const uint64_t *s, const double *c, int cap, int l,
                   int inv, double *v) {
  return gpk_impl<double>(nd, s, c, cap, l, inv, v);
}
int mgrref_gpk_f32(int nd, const uint64_t *s, const double *c, int cap, int l,
                   int inv, float *v) {
  return gpk_impl<float>(nd, s, c, cap, l, inv, v);
}
int mgrref_masstrans_f64(int nd, const uint64_t *s, const double *c, int cap,
                         int l, int dim, const double *in, double *out,
                         int fused, double *coef) {
  return masstrans_impl<double>(nd, s, c, cap, l, dim, in, out, fused, coef);
}
int mgrref_masstrans_f32(int nd, const uint64_t *s, const double *c, int cap,
                         int l, int dim, const float *in, float *out, int fused,
                         float *coef) {
  return masstrans_impl<float>(nd, s, c, cap, l, dim, in, out, fused, coef);
}
int mgrref_solve_f64(int nd, const uint64_t *s, const double *c, int cap, int l,
                     int dim, double *f) {
  return solve_impl<double>(nd, s, c, cap, l, dim, f);
}
int mgrref_solve_f32(int nd, const uint64_t *s, const double *c, int cap, int l,
                     int dim, float *f) {
  return solve_impl<float>(nd, s, c, cap, l, dim, f);
}

// embarrassing_decompose (parallel_impl.hpp:810-847) + recompose of every
// block, each block an independent 3-D grid of the same shape; `workers`
// threads.  Used by bench.py --impl reference to time the reference on all
// host cores.  values/classes: nblocks * N elements back to back.
int mgrref_embarrassing_roundtrip_coords_f32(int nd, const uint64_t *shape, int nblocks,
                                             int workers, const double *coords,
                                             const float *values, float *classes,
                                             float *recomposed, double *t_dec,
                                             double *t_rec);

int mgrref_embarrassing_roundtrip_f32(int nd, const uint64_t *shape,
                                      int nblocks, int workers,
                                      const float *values, float *classes,
                                      float *recomposed, double *t_dec,
                                      double *t_rec) {
  return mgrref_embarrassing_roundtrip_coords_f32(nd, shape, nblocks, workers, nullptr, values,
                                                  classes, recomposed, t_dec, t_rec);
}

// The same with per-block coordinates (`coords`: nblocks consecutive
// sets of sum(shape) doubles, e.g. slices of a larger field's global
// coordinates; NULL = uniform_coords per block).
int mgrref_embarrassing_roundtrip_coords_f32(int nd, const uint64_t *shape, int nblocks,
                                             int workers, const double *coords,
                                             const float *values, float *classes,
                                             float *recomposed, double *t_dec,
                                             double *t_rec) {
  try {
    const mgr::Shape s = to_shape(nd, shape);
    const std::size_t n = mgr::num_elements(s);
    std::size_t csum = 0;
    for (int d = 0; d < nd; ++d)
      csum += shape[d];
    std::vector<mgr::TensorGrid<float>> blocks(nblocks);
    for (int b = 0; b < nblocks; ++b) {
      blocks[b].shape = s;
      blocks[b].coords = to_coords(nd, shape, coords ? coords + b * csum : nullptr);
      blocks[b].values.assign(values + b * n, values + (b + 1) * n);
    }
    const auto t0 = std::chrono::steady_clock::now();
    const auto out = mgr::embarrassing_decompose(blocks, workers);
    const auto t1 = std::chrono::steady_clock::now();
    // recompose: the reference has no parallel recompose driver; use the
    // same pool shape (one std::thread per worker, blocks dealt in order).
    std::vector<std::thread> th;
    std::vector<mgr::TensorGrid<float>> rec(nblocks);
    const int pool = std::max(1, std::min(workers, nblocks));
    for (int w = 0; w < pool; ++w)
      th.emplace_back([&, w] {
        for (int b = w; b < nblocks; b += pool)
          rec[b] = mgr::recompose(out[b], out[b].levels);
      });
    for (auto &t : th)
      t.join();
    const auto t2 = std::chrono::steady_clock::now();
    for (int b = 0; b < nblocks; ++b) {
      std::size_t off = b * n;
      for (const auto &c : out[b].classes) {
        if (classes)
          std::memcpy(classes + off, c.data(), c.size() * sizeof(float));
        off += c.size();
      }
      if (recomposed)
        std::memcpy(recomposed + b * n, rec[b].values.data(), n * sizeof(float));
    }
    *t_dec = std::chrono::duration<double>(t1 - t0).count();
    *t_rec = std::chrono::duration<double>(t2 - t1).count();
    return 0;
  } catch (const mgr::Error &e) {
    return code_of(e);
  } catch (...) {
    return 15;
  }
}

// Deterministic test data exactly as the reference tests generate it
// (tests/oracle.cpp:167-186).
void mgrref_random_vector(uint64_t n, unsigned seed, double lo, double hi,
                          double *out) {
  const auto v = oracle::random_vector(n, seed, lo, hi);
  std::memcpy(out, v.data(), n * sizeof(double));
}
void mgrref_random_increasing_coords(uint64_t n, unsigned seed, double *out) {
  const auto v = oracle::random_increasing_coords(n, seed);
  std::memcpy(out, v.data(), n * sizeof(double));
}

int64_t mgrref_write_refactored_f32(int nd, const uint64_t *shape, const double *coords,
                                    int levels, const float *classes, const char *path) {
  return write_impl<float>(nd, shape, coords, levels, classes, path);
}
int64_t mgrref_write_refactored_f64(int nd, const uint64_t *shape, const double *coords,
                                    int levels, const double *classes, const char *path) {
  return write_impl<double>(nd, shape, coords, levels, classes, path);
}
// read_refactored (pipeline.cpp:233-300): classes 0..k (k < 0: all) into a
// flat buffer; returns bytes consumed, or -(status code).
int64_t mgrref_read_refactored(const char *path, int k, void *classes, int *loaded) {
  try {
    std::optional<std::size_t> want;
    if (k >= 0)
      want = std::size_t(k);
    const auto rr = mgr::read_refactored(path, want);
    std::size_t off = 0;
    std::visit(
        [&](const auto &r) {
          using Real = typename std::decay_t<decltype(r.classes[0])>::value_type;
          for (const auto &c : r.classes) {
            std::memcpy(static_cast<Real *>(classes) + off, c.data(), c.size() * sizeof(Real));
            off += c.size();
          }
        },
        rr.data);
    if (loaded)
      *loaded = int(rr.classes_loaded);
    return int64_t(rr.bytes_consumed);
  } catch (const mgr::Error &e) {
    return -int64_t(code_of(e));
  } catch (...) {
    return -15;
  }
}
int64_t mgrref_compress_f32(int nd, const uint64_t *shape, const double *coords,
                            const float *values, double eb, int codec, uint8_t *out,
                            uint64_t cap, double *bin, double *measured) {
  return compress_impl<float>(nd, shape, coords, values, eb, codec, out, cap, bin, measured);
}
int64_t mgrref_compress_f64(int nd, const uint64_t *shape, const double *coords,
                            const double *values, double eb, int codec, uint8_t *out,
                            uint64_t cap, double *bin, double *measured) {
  return compress_impl<double>(nd, shape, coords, values, eb, codec, out, cap, bin, measured);
}
// decompress into a flat value buffer; returns 0 or -(status code)
int64_t mgrref_decompress(const uint8_t *bytes, uint64_t n, void *values, uint64_t cap_elems) {
  try {
    const auto d = mgr::decompress(std::span<const uint8_t>(bytes, n));
    int64_t rc = 0;
    std::visit(
        [&](const auto &g) {
          using Real = typename std::decay_t<decltype(g.values)>::value_type;
          if (g.values.size() > cap_elems) {
            rc = -16;
            return;
          }
          std::memcpy(values, g.values.data(), g.values.size() * sizeof(Real));
        },
        d.grid);
    return rc;
  } catch (const mgr::Error &e) {
    return -int64_t(code_of(e));
  } catch (...) {
    return -15;
  }
}
// PassStats of the reference engine (refactor.hpp:223-421): decompose of the
// given f64 grid (levels cap 0 = full), then -- when `recompose` -- a full
// recompose into the SAME stats object (it appends without clearing).  Per
// level record (finest first for the decompose part): level, elements,
// coefficient in/out, fused_copy in/out, then nd x (masstrans in, out),
// nd x (solve in, out), apply in/out = 8 + 4 nd words.  *nlevels = records.
int mgrref_pass_stats_f64(int nd, const uint64_t *shape, const double *coords, int levels_cap,
                          const double *values, int recompose, uint64_t *out, int cap_records,
                          int *nlevels) {
  try {
    mgr::TensorGrid<double> g;
    g.shape = to_shape(nd, shape);
    g.coords = to_coords(nd, shape, coords);
    g.values.assign(values, values + mgr::num_elements(g.shape));
    mgr::PassStats st;
    mgr::RefactorOptions opt;
    if (levels_cap > 0)
      opt.levels = std::size_t(levels_cap);
    opt.stats = &st;
    const auto r = mgr::decompose(g, opt);
    if (recompose)
      (void)mgr::recompose(r, r.levels, opt);
    *nlevels = int(st.levels.size());
    const std::size_t w = 8 + 4 * std::size_t(nd);
    for (std::size_t i = 0; i < st.levels.size() && int(i) < cap_records; ++i) {
      const auto &lv = st.levels[i];
      uint64_t *o = out + i * w;
      o[0] = lv.level;
      o[1] = lv.level_elements;
      o[2] = lv.coefficient.in;
      o[3] = lv.coefficient.out;
      o[4] = lv.fused_copy.in;
      o[5] = lv.fused_copy.out;
      for (int d = 0; d < nd; ++d) {
        o[6 + 2 * d] = lv.masstrans[d].in;
        o[7 + 2 * d] = lv.masstrans[d].out;
        o[6 + 2 * nd + 2 * d] = lv.solve[d].in;
        o[7 + 2 * nd + 2 * d] = lv.solve[d].out;
      }
      o[6 + 4 * nd] = lv.apply.in;
      o[7 + 4 * nd] = lv.apply.out;
    }
    return 0;
  } catch (const mgr::Error &e) {
    return code_of(e);
  } catch (...) {
    return 15;
  }
}

// mgr::weighted_l2_norm (grid.hpp:218-244) of an f64 grid.
double mgrref_weighted_l2_norm_f64(int nd, const uint64_t *shape, const double *coords,
                                   const double *values) {
  mgr::TensorGrid<double> g;
  g.shape = to_shape(nd, shape);
  g.coords = to_coords(nd, shape, coords);
  g.values.assign(values, values + mgr::num_elements(g.shape));
  return mgr::weighted_l2_norm(g);
}

// CommReport::to_json (parallel.cpp:264-292) of a report built from plain
// fields: phases as (name, messages, elements, local, seconds), idle records
// as (level, dim, stages, counts...).  Writes at most cap bytes (NUL-ended).
int mgrref_comm_report_json(int workers, int scheme, uint64_t grid_elements, int nphases,
                            const char *const *names, const uint64_t *counts,
                            const double *seconds, int nidle, const uint64_t *idle_words,
                            char *out, uint64_t cap) {
  mgr::CommReport rep;
  rep.workers = workers;
  rep.scheme = scheme ? mgr::PartitionScheme::shifted_round_robin : mgr::PartitionScheme::block;
  rep.total_grid_elements = grid_elements;
  for (int i = 0; i < nphases; ++i) {
    auto &ph = rep.phases[names[i]];
    ph.messages = counts[3 * i];
    ph.elements = counts[3 * i + 1];
    ph.local_elements = counts[3 * i + 2];
    ph.seconds = seconds[i];
  }
  const uint64_t *w = idle_words;
  for (int i = 0; i < nidle; ++i) {
    mgr::IdleRecord rec;
    rec.level = w[0];
    rec.dim = w[1];
    for (uint64_t k = 0; k < w[2]; ++k)
      rec.idle_per_stage.push_back(int(w[3 + k]));
    w += 3 + w[2];
    rep.idle.push_back(std::move(rec));
  }
  const std::string j = rep.to_json();
  if (j.size() + 1 > cap)
    return 3;
  std::memcpy(out, j.c_str(), j.size() + 1);
  return 0;
}

uint32_t mgrref_crc32(const uint8_t *data, uint64_t n) {
  return mgr::crc32(std::span<const uint8_t>(data, n));
}

} // extern "C"
