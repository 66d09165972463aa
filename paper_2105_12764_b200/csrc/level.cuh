// level.cuh -- per-level geometry handed to the kernels by value.
//
// Every grid is processed as 3-D: user dimensions keep their order and
// missing ones are padded with extent 1.  An extent-1 (or 2) dimension never
// refines, its class-type extents are 0 for the "fine" bit, so the class
// order of the padded grid is exactly the reference's (grid.cpp:140-165).
#pragma once

#include <cstdint>

namespace mgrg {

template <typename R> struct LevelGeom {
  uint32_t n[3];        // level-l extents (the lattice being processed)
  uint32_t m[3];        // level-(l-1) extents (coarse lattice)
  uint32_t refine;      // bit d set: dimension d refines at this level
  const R *h[3];        // level-l spacings along d, n[d]-1 values (grid.cpp:60-65)
  const R *r[3];        // level-l ratios along d, n[d]-2 values (grid.cpp:66-71)
  uint64_t tbase[8];    // class type base per mask (grid.cpp:151-162)
  uint32_t tex[8];      // class type extent along dim 0 per mask
  uint32_t tey[8];      // class type extent along dim 1 per mask

  __host__ __device__ uint64_t nodes() const {
    return uint64_t(n[0]) * n[1] * n[2];
  }
  __host__ __device__ uint64_t coarse_nodes() const {
    return uint64_t(m[0]) * m[1] * m[2];
  }
};

// Thomas factors of one dimension of the level-(l-1) lattice
// (TridiagonalOperator::build, kernels.hpp:107-135), working precision.
template <typename R> struct ThomasGeom {
  const R *h;   // m-1 spacings
  const R *fwd; // m forward multipliers (fwd[0] = 0)
  const R *ip;  // m reciprocal pivots
  uint32_t m;
};

// Epilogue of the last solve of a level (refactor.hpp:380-422):
//   none: the solution z stays in f;
//   add : out[i] = base[i] + z[i]   (decompose apply_pack);
//   sub : out[i] = base[i] - z[i]   (recompose unapply_expand).
enum class Epi : int { none = 0, add = 1, sub = 2 };

} // namespace mgrg
