/*
 * mgr_oracle.h -- CPU restatement of the reference decompose/recompose path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker the parity tests, smoke()
 * and bench.py's cpu_baseline leg compare the CUDA path against.  Nothing in
 * the product (paper_2105_12764_b200/, include/) may link or call it.
 *
 * Parity pinned: tests/test_oracle.py checks every function here bit-for-bit
 * against the reference itself compiled from /root/reference by
 * oracle/Makefile (oracle/_ref/libmgr_ref.so) and against the golden vectors
 * of the reference's own tests (tests/golden/).
 *
 * Every function restates the reference algorithm in plain C with the same
 * floating-point evaluation order (no FMA contraction: build with
 * -ffp-contract=off), so results are bit-identical.  Citations are
 * /root/reference/proj/<file>:<line>.
 *
 * Conventions (shared with include/mgrg.h):
 *   - shape[d], d = 0..ndims-1, row-major with dimension 0 fastest
 *     (ndarray.hpp:16-26);
 *   - coords: NULL for uniform i/(n-1) coordinates (grid.cpp:7-12), else the
 *     per-dimension coordinate arrays concatenated, dimension 0 first;
 *   - levels_cap: 0 = full depth, else RefactorOptions::levels
 *     (refactor.hpp:71-76);
 *   - classes: ONE buffer of N elements, class l at offset N_{l-1}
 *     (class 0 = coarsest nodal values at offset 0).
 * Return value: 0 on success, else an MGRG_* status code (include/mgrg.h).
 */
#ifndef MGR_ORACLE_H
#define MGR_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Hierarchy depth and per-level extents: level_extents[l*ndims + d]
 * (capacity (64+1)*ndims).  grid.cpp:78-112, min_extent as passed. */
int mgro_hierarchy(int ndims, const uint64_t *shape, const double *coords,
                   int levels_cap, int min_extent, int *levels_out,
                   uint64_t *level_extents);

/* Offsets of classes 0..L in the single class buffer plus the total:
 * offsets[0..L+1] (offsets[l] = N_{l-1}, offsets[0] = 0, offsets[L+1] = N). */
int mgro_class_offsets(int ndims, const uint64_t *shape, int levels,
                       uint64_t *offsets);

/* Class layout of one level (grid.cpp:140-165): type_base[mask],
 * type_extents[mask*ndims + d] for mask in [0, 2^ndims). */
int mgro_class_layout(int ndims, const uint64_t *shape, int levels, int level,
                      uint64_t *type_base, uint64_t *type_extents);

/* Full decompose / recompose (refactor.hpp:159-204, 462-496). */
int mgro_decompose_f64(int ndims, const uint64_t *shape, const double *coords,
                       int levels_cap, const double *values, double *classes,
                       int *levels_out);
int mgro_decompose_f32(int ndims, const uint64_t *shape, const double *coords,
                       int levels_cap, const float *values, float *classes,
                       int *levels_out);
int mgro_recompose_f64(int ndims, const uint64_t *shape, const double *coords,
                       int levels, const double *classes, int classes_used,
                       double *values);
int mgro_recompose_f32(int ndims, const uint64_t *shape, const double *coords,
                       int levels, const float *classes, int classes_used,
                       float *values);

/* Unit-level kernels on the full-depth hierarchy (levels_cap applies).
 * compute/restore_coefficients: in place on a packed level-`level` array
 * (kernels.hpp:284-310). */
int mgro_gpk_f64(int ndims, const uint64_t *shape, const double *coords,
                 int levels_cap, int level, int inverse, double *values);
int mgro_gpk_f32(int ndims, const uint64_t *shape, const double *coords,
                 int levels_cap, int level, int inverse, float *values);

/* masstrans_apply (kernels.hpp:328-412): `in` has masstrans_input_shape
 * extents, `out` the same with dim reduced; fused_copy writes the class
 * (class order) into coef_out (dim 0 only). */
int mgro_masstrans_f64(int ndims, const uint64_t *shape, const double *coords,
                       int levels_cap, int level, int dim, const double *in,
                       double *out, int fused_copy, double *coef_out);
int mgro_masstrans_f32(int ndims, const uint64_t *shape, const double *coords,
                       int levels_cap, int level, int dim, const float *in,
                       float *out, int fused_copy, float *coef_out);

/* solve_correction (kernels.hpp:417-448): in place on the level-(l-1)
 * lattice. */
int mgro_solve_f64(int ndims, const uint64_t *shape, const double *coords,
                   int levels_cap, int level, int dim, double *f);
int mgro_solve_f32(int ndims, const uint64_t *shape, const double *coords,
                   int levels_cap, int level, int dim, float *f);

/* reorder (grid.hpp:177-196): direction 0 = to_hierarchical, 1 = natural. */
int mgro_reorder_f64(int ndims, const uint64_t *shape, const double *coords,
                     int levels_cap, int level, int direction,
                     const double *in, double *out);

/* Worker threads of the engine's row-parallel loops (0 = all online CPUs,
 * 1 = serial); returns the previous setting.  Never changes a value. */
int mgro_set_threads(int n);

#ifdef __cplusplus
}
#endif

#endif
