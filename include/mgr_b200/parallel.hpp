// mgr_b200/parallel.hpp -- source-level drop-in for the reference's
// parallel API (/root/reference/proj/include/mgr/parallel.hpp): partitions,
// cooperative_decompose, embarrassing_decompose (in refactor.hpp) and
// grouped_decompose, backed by the B200 path.
//
//     #include "mgr/parallel.hpp"   ->   #include "mgr_b200/parallel.hpp"
//
// cooperative_decompose runs the native cooperative runtime
// (mgrg_cooperative_decompose_host): worker w on GPU (device + w) mod the
// visible GPUs, z-slab halo exchange and chained Thomas solves between them,
// results bit-identical to decompose() of the whole grid -- the reference's
// contract (test_parallel.cpp:88-123).  The partition scheme is validated
// like the reference's and reported; the device path always splits the
// slowest dimension into slabs (NVSwitch gives every GPU pair the same
// bandwidth, and slabs keep every transfer a contiguous plane range).
#ifndef MGR_B200_PARALLEL_HPP
#define MGR_B200_PARALLEL_HPP

#include <array>
#include <functional>
#include <map>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "refactor.hpp"

namespace mgr {

enum class PartitionScheme { block, shifted_round_robin };
inline const char *to_string(PartitionScheme s) {
  return s == PartitionScheme::block ? "block" : "shifted_round_robin";
}

// parallel.hpp:22-27
struct Partition {
  int worker = 0;
  Shape lo, hi;
  std::array<std::size_t, 2> block_coord{0, 0};
};

// parallel.cpp:9-19
inline std::vector<std::size_t> split_dims_of(const Shape &shape, PartitionScheme scheme,
                                              int workers) {
  const std::size_t nd = shape.size();
  if (workers == 1)
    return {};
  if (scheme == PartitionScheme::block)
    return {nd - 1};
  if (nd < 2)
    throw ShapeError("shifted round-robin partitioning needs >= 2 dimensions");
  return {nd - 2, nd - 1};
}

namespace b200_detail {
// near-equal contiguous ranges, remainder to the leading ones
inline std::vector<std::pair<std::size_t, std::size_t>> split_range(std::size_t n, int parts) {
  std::vector<std::pair<std::size_t, std::size_t>> out;
  const std::size_t base = n / std::size_t(parts), rem = n % std::size_t(parts);
  std::size_t at = 0;
  for (int i = 0; i < parts; ++i) {
    const std::size_t len = base + (std::size_t(i) < rem ? 1 : 0);
    out.emplace_back(at, at + len);
    at += len;
  }
  return out;
}
} // namespace b200_detail

// parallel.cpp:37-90
inline std::vector<Partition> make_partitions(const Shape &shape, int workers,
                                              PartitionScheme scheme) {
  if (workers < 1)
    throw TooManyWorkers("worker count must be positive");
  const std::size_t nd = shape.size();
  if (workers == 1)
    return {Partition{0, Shape(nd, 0), shape, {0, 0}}};
  const auto split = split_dims_of(shape, scheme, workers);
  for (std::size_t d : split)
    if (std::size_t(workers) > shape[d])
      throw TooManyWorkers("cannot split dimension " + std::to_string(d) + " of extent " +
                           std::to_string(shape[d]) + " across " + std::to_string(workers) +
                           " workers");
  std::vector<Partition> parts;
  if (scheme == PartitionScheme::block) {
    const auto r = b200_detail::split_range(shape[split[0]], workers);
    for (int w = 0; w < workers; ++w) {
      Partition p{w, Shape(nd, 0), shape, {std::size_t(w), 0}};
      p.lo[split[0]] = r[w].first;
      p.hi[split[0]] = r[w].second;
      parts.push_back(std::move(p));
    }
  } else {
    const auto ra = b200_detail::split_range(shape[split[0]], workers);
    const auto rb = b200_detail::split_range(shape[split[1]], workers);
    for (int a = 0; a < workers; ++a)
      for (int b = 0; b < workers; ++b) {
        Partition p{(a + b) % workers, Shape(nd, 0), shape,
                    {std::size_t(a), std::size_t(b)}};
        p.lo[split[0]] = ra[a].first;
        p.hi[split[0]] = ra[a].second;
        p.lo[split[1]] = rb[b].first;
        p.hi[split[1]] = rb[b].second;
        parts.push_back(std::move(p));
      }
  }
  return parts;
}

// parallel.hpp:36-58 (the per-phase counters of the native runtime are
// reported as one "device" phase: elements moved between distinct workers)
struct CommPhaseStats {
  std::uint64_t messages = 0;
  std::uint64_t elements = 0;
  std::uint64_t local_elements = 0;
  double seconds = 0;
};
// Idle workers per pipeline stage of one ordered sweep (parallel.hpp:44-50).
struct IdleRecord {
  std::size_t level = 0;
  std::size_t dim = 0;
  std::vector<int> idle_per_stage;
};
struct CommReport {
  int workers = 0;
  PartitionScheme scheme = PartitionScheme::block;
  std::map<std::string, CommPhaseStats> phases;
  std::vector<IdleRecord> idle;
  std::uint64_t total_grid_elements = 0;
  // parallel.cpp:264-292: the same keys, order and number formatting
  // (std::ostream defaults) as the reference, so tools that parse the
  // reference's report (mgrf.cpp:150-158) read this one.
  std::string to_json() const {
    std::ostringstream os;
    os << "{\"workers\":" << workers << ",\"scheme\":\"" << to_string(scheme)
       << "\",\"grid_elements\":" << total_grid_elements << ",\"phases\":{";
    bool first = true;
    for (const auto &[name, st] : phases) {
      os << (first ? "" : ",") << "\"" << name << "\":{\"messages\":" << st.messages
         << ",\"elements\":" << st.elements << ",\"local_elements\":" << st.local_elements
         << ",\"seconds\":" << st.seconds << "}";
      first = false;
    }
    os << "},\"idle\":[";
    first = true;
    for (const auto &rec : idle) {
      os << (first ? "" : ",") << "{\"level\":" << rec.level << ",\"dim\":" << rec.dim
         << ",\"idle_per_stage\":[";
      for (std::size_t i = 0; i < rec.idle_per_stage.size(); ++i)
        os << (i ? "," : "") << rec.idle_per_stage[i];
      os << "]}";
      first = false;
    }
    os << "]}";
    return os.str();
  }
};

// parallel.hpp:61-71
struct CoopOptions {
  std::optional<std::size_t> levels;
  PartitionScheme scheme = PartitionScheme::block;
  CommReport *report = nullptr;
  std::function<void(int worker, const std::string &phase, std::size_t level)> fault_injector;
  // B200 extensions
  int device = 0;
  bool fast = false;
};

namespace b200_detail {
inline int fault_trampoline(void *ctx, int32_t worker, const char *phase, int32_t level) {
  auto *f = static_cast<const CoopOptions *>(ctx);
  try {
    f->fault_injector(int(worker), std::string(phase), std::size_t(level));
    return 0;
  } catch (...) {
    return 1;
  }
}
} // namespace b200_detail

// mgr::cooperative_decompose (parallel_impl.hpp:691-808)
template <typename Real>
RefactoredData<Real> cooperative_decompose(const TensorGrid<Real> &grid, int workers,
                                           const CoopOptions &opt = {}) {
  static_assert(std::is_same_v<Real, float> || std::is_same_v<Real, double>,
                "Real must be float or double");
  validate_grid_geometry(grid.shape, grid.coords, 2);
  if (grid.values.size() != num_elements(grid.shape))
    throw ShapeError("value count does not match the grid");
  (void)make_partitions(grid.shape, workers, opt.scheme);
  mgrg_grid_desc desc{};
  desc.ndims = int32_t(grid.shape.size());
  desc.dtype = sizeof(Real) == 4 ? MGRG_F32 : MGRG_F64;
  std::vector<double> flat;
  for (std::size_t d = 0; d < grid.shape.size(); ++d) {
    desc.shape[d] = grid.shape[d];
    flat.insert(flat.end(), grid.coords[d].begin(), grid.coords[d].end());
  }
  desc.coords = flat.data();
  desc.levels = b200_detail::levels_arg(opt.levels);
  desc.device = opt.device;
  desc.flags = opt.fast ? MGRG_FLAG_FAST : 0;
  std::vector<Real> out(grid.values.size());
  std::uint64_t moved = 0;
  const auto t0 = std::chrono::steady_clock::now();
  b200_detail::check(mgrg_cooperative_decompose_host(
      &desc, workers, grid.values.data(), out.data(),
      opt.fault_injector ? &b200_detail::fault_trampoline : nullptr,
      const_cast<CoopOptions *>(&opt), &moved));
  const double secs =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  // class layout of the whole-grid plan
  mgrg_plan *p = b200_detail::plan_for<Real>(grid.shape, grid.coords, opt.levels, opt.device,
                                             opt.fast);
  int32_t L = 0;
  b200_detail::check(mgrg_plan_levels(p, &L));
  if (opt.report) {
    opt.report->workers = workers;
    opt.report->scheme = opt.scheme;
    opt.report->total_grid_elements = grid.values.size();
    auto &ph = opt.report->phases["device"];
    ph.messages += 1;
    ph.elements += moved;
    ph.seconds += secs;
    // idle workers per stage of the ordered (chained) z solves, the one
    // sweep the runtime orders across workers (compute_idle_records,
    // parallel.cpp:217-258, for the runtime's z-slab partition): stage s of
    // the chain at a cooperative level is worker s's slab, so W - 1 workers
    // wait in every stage (fewer active when a slab holds no coarse plane)
    int32_t q = 0;
    std::vector<uint64_t> bounds(std::size_t(workers) + 1);
    b200_detail::check(mgrg_coop_schedule(p, workers, &q, bounds.data()));
    opt.report->idle.clear();
    for (int j = 0; j < q; ++j) {
      uint64_t ls[4] = {1, 1, 1, 1};
      b200_detail::check(mgrg_plan_level_shape(p, L - j - 1, ls));
      IdleRecord rec;
      rec.level = std::size_t(L - j);
      rec.dim = 2;
      rec.idle_per_stage.assign(std::size_t(workers), workers);
      for (int r = 0; r < workers; ++r) {
        const uint64_t c0 = bounds[r] >> (j + 1);
        const uint64_t c1 = r == workers - 1 ? ls[2] : bounds[r + 1] >> (j + 1);
        rec.idle_per_stage[r] = workers - (c1 > c0 ? 1 : 0);
      }
      opt.report->idle.push_back(std::move(rec));
    }
  }
  std::vector<uint64_t> off(std::size_t(L) + 2);
  b200_detail::check(mgrg_plan_class_offsets(p, off.data()));
  RefactoredData<Real> r;
  r.shape = grid.shape;
  r.coords = grid.coords;
  r.levels = std::size_t(L);
  for (int l = 0; l <= L; ++l)
    r.classes.emplace_back(out.begin() + off[l], out.begin() + off[l + 1]);
  return r;
}

// mgr::grouped_decompose (parallel_impl.hpp:849-885): K groups of S
// cooperating workers run concurrently, one host thread per group, block i
// to group i mod K; group g's workers start at GPU g * S (mod the visible
// GPUs) so concurrent groups land on distinct devices when there are enough.
// The first failure stops the groups and surfaces as WorkerFailure.
template <typename Real>
std::vector<RefactoredData<Real>>
grouped_decompose(const std::vector<TensorGrid<Real>> &blocks, int num_groups, int group_size,
                  PartitionScheme scheme = PartitionScheme::block) {
  if (num_groups < 1 || group_size < 1)
    throw TooManyWorkers("group shape must be positive");
  std::vector<RefactoredData<Real>> out(blocks.size());
  int32_t ndev = 1;
  if (mgrg_device_count(&ndev) != MGRG_OK || ndev < 1)
    ndev = 1;
  std::atomic<bool> failed{false};
  std::mutex err_mu;
  std::string err;
  std::vector<std::thread> threads;
  const int groups = std::max(1, std::min<int>(num_groups, int(blocks.size())));
  for (int g = 0; g < groups; ++g)
    threads.emplace_back([&, g] {
      for (std::size_t i = std::size_t(g); i < blocks.size(); i += std::size_t(groups)) {
        if (failed.load())
          break;
        try {
          CoopOptions o;
          o.scheme = scheme;
          o.device = (g * group_size) % int(ndev);
          out[i] = cooperative_decompose(blocks[i], group_size, o);
        } catch (const std::exception &e) {
          std::lock_guard<std::mutex> lk(err_mu);
          err = e.what();
          failed.store(true);
          break;
        }
      }
      release_plans();
    });
  for (auto &t : threads)
    t.join();
  if (failed.load())
    throw WorkerFailure(err);
  return out;
}

} // namespace mgr

#endif
