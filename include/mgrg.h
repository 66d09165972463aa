/*
 * mgrg.h -- C ABI of the B200-native multigrid refactoring path.
 *
 * This is the binary drop-in boundary under the reference's C++ entry points
 * (/root/reference/proj/include/mgr/refactor.hpp).  The reference's public
 * API is header-only templates, so the source-level drop-in is
 * include/mgr_b200/refactor.hpp (namespace mgr, same names/types), which calls
 * the functions below; ctypes / cgo-style bindings call them directly.
 *
 * Layout conventions (identical to the reference):
 *   - values: row-major, dimension 0 fastest (ndarray.hpp:16-26);
 *   - classes: ONE buffer of N elements; class 0 (coarsest nodal values,
 *     packed row-major) at offset 0, class l (level-l coefficients in class
 *     order, grid.hpp:136-164) at offset N_{l-1} = number of level-(l-1)
 *     nodes.  This equals the concatenation of RefactoredData::classes
 *     (refactor.hpp:18-32) and the MGRF payload order (pipeline.cpp:197-200);
 *   - coords: NULL for uniform coordinates i/(n-1) (grid.cpp:7-12), else the
 *     per-dimension coordinate arrays concatenated, dimension 0 first.
 *
 * Numerics: every kernel evaluates the reference's expressions in the same
 * order with IEEE round-to-nearest and no FMA contraction, so classes and
 * reconstructions are bit-identical to the reference CPU path.
 *
 * Threading: a plan owns its device workspace and must not be used by two
 * calls concurrently; distinct plans are independent.  The last
 * error message is thread-local.
 *
 * Errors: every function returns an mgrg_status; the codes map 1:1 onto the
 * reference's exception types (errors.hpp:27-37).
 */
#ifndef MGRG_H
#define MGRG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum mgrg_status {
  MGRG_OK = 0,
  MGRG_INVALID_GRID = 1,      /* mgr::InvalidGrid    (grid.cpp:17-34)        */
  MGRG_INVALID_LEVEL = 2,     /* mgr::InvalidLevel   (refactor.hpp:480-482)  */
  MGRG_SHAPE_ERROR = 3,       /* mgr::ShapeError     (grid.hpp:44-47)        */
  MGRG_INVALID_FUSION = 4,    /* mgr::InvalidFusion  (kernels.hpp:337-338)   */
  MGRG_SINGULAR_SYSTEM = 5,   /* mgr::SingularSystem (kernels.hpp:121-131)   */
  MGRG_TOO_MANY_WORKERS = 6,  /* mgr::TooManyWorkers                         */
  MGRG_WORKER_FAILURE = 7,    /* mgr::WorkerFailure  (parallel_impl.hpp:845) */
  MGRG_CORRUPT_FILE = 8,      /* mgr::CorruptFile                            */
  MGRG_MISSING_CLASS = 9,     /* mgr::MissingClass   (refactor.hpp:483-485)  */
  MGRG_INVALID_BOUND = 10,    /* mgr::InvalidBound                           */
  MGRG_IO_ERROR = 11,         /* mgr::IoError                                */
  MGRG_CUDA_ERROR = 12,       /* device failure (no reference equivalent)   */
  MGRG_NCCL_ERROR = 13,       /* collective failure                          */
  MGRG_UNSUPPORTED = 14,      /* a limit of this implementation (extent > 2^31) */
  MGRG_INVALID_ARGUMENT = 15, /* null pointer, bad dtype, ...                */
  MGRG_OUT_OF_MEMORY = 16
} mgrg_status;

typedef enum mgrg_dtype { MGRG_F32 = 4, MGRG_F64 = 8 } mgrg_dtype;

/* Grid description: TensorGrid minus the values (grid.hpp:19-26) plus
 * RefactorOptions::levels (refactor.hpp:71-76). */
typedef struct mgrg_grid_desc {
  int32_t ndims;         /* 1..4 (ndarray.hpp:12 kMaxDims)                  */
  int32_t dtype;         /* mgrg_dtype */
  uint64_t shape[4];     /* finest-level extents, dim 0 fastest */
  const double *coords;  /* NULL = uniform; else sum(shape) doubles */
  int32_t levels;        /* 0 = full depth, else the RefactorOptions cap */
  int32_t device;        /* CUDA device ordinal the plan lives on */
  int32_t flags;         /* MGRG_FLAG_* */
} mgrg_grid_desc;

/* Arithmetic policy.  Default: every kernel evaluates the reference's
 * expressions in the reference's order with no FMA contraction, so results
 * are bit-identical to the reference CPU path.  MGRG_FLAG_FAST: interpolation
 * as one FMA and the merged mass-trans as precomputed 5-tap FMA chains
 * (same operator; results differ at rounding level, range-normalized
 * ~1e-7 f32 / ~1e-16 f64). */
#define MGRG_FLAG_FAST 1

typedef struct mgrg_plan mgrg_plan;

/* Plan = build_hierarchy (grid.cpp:78-112) with min_extent 2 as decompose
 * validates it (refactor.hpp:465-466), per-level class layouts
 * (grid.cpp:140-165), Thomas factors built in the working precision
 * (kernels.hpp:107-135), geometry uploaded to the device, and the device
 * workspace (about N/4 elements).  All allocation happens here. */
mgrg_status mgrg_plan_create(const mgrg_grid_desc *desc, mgrg_plan **plan);
mgrg_status mgrg_plan_destroy(mgrg_plan *plan);

/* Hierarchy depth L (RefactoredData::levels). */
mgrg_status mgrg_plan_levels(const mgrg_plan *plan, int32_t *levels);
/* offsets[0..L+1]: class l occupies [offsets[l], offsets[l+1]); offsets[0]=0,
 * offsets[L+1] = N. */
mgrg_status mgrg_plan_class_offsets(const mgrg_plan *plan, uint64_t *offsets);
/* Level-l extents, ndims entries (GridHierarchy::level_shape). */
mgrg_status mgrg_plan_level_shape(const mgrg_plan *plan, int32_t level,
                                  uint64_t *extents);
/* Total element count N and device workspace bytes owned by the plan. */
mgrg_status mgrg_plan_sizes(const mgrg_plan *plan, uint64_t *num_elements,
                            uint64_t *workspace_bytes);

/* ---- whole-path entry points (device buffers) --------------------------
 * mgr::decompose (refactor.hpp:462-474): d_values (N elements, not
 * modified) -> d_classes (N elements, class layout above).  Asynchronous on
 * `stream` (a cudaStream_t; NULL = legacy default stream). */
mgrg_status mgrg_decompose(mgrg_plan *plan, const void *d_values,
                           void *d_classes, void *stream);

/* mgr::recompose (refactor.hpp:476-496): classes 0..classes_used are read,
 * classes above it are treated as zero (never read).  classes_used > L ->
 * MGRG_INVALID_LEVEL. */
mgrg_status mgrg_recompose(mgrg_plan *plan, const void *d_classes,
                           int32_t classes_used, void *d_values, void *stream);

/* ---- host-buffer entry points (what the reference's callers pass) -------
 * Same semantics; host -> device copy, the device path, device -> host copy,
 * synchronous.  Pinned host memory (cudaHostAlloc / cudaHostRegister) is
 * DMA'd directly; pageable memory streams through plan-owned pinned rings
 * with multi-threaded host copies overlapping the DMA and the kernels. */
mgrg_status mgrg_decompose_host(mgrg_plan *plan, const void *h_values,
                                void *h_classes);
mgrg_status mgrg_recompose_host(mgrg_plan *plan, const void *h_classes,
                                int32_t classes_used, void *h_values);
/* The same with the classes in separate host buffers, one per class, as
 * RefactoredData::classes holds them (refactor.hpp:18-30): h_classes[l]
 * points to class l's nodes (offsets[l+1] - offsets[l] elements of
 * mgrg_plan_class_offsets), l = 0..L for decompose, 0..classes_used for
 * recompose (others are not read).  No flat concatenation is made. */
mgrg_status mgrg_decompose_host_classes(mgrg_plan *plan, const void *h_values,
                                        void *const *h_classes);
mgrg_status mgrg_recompose_host_classes(mgrg_plan *plan, const void *const *h_classes,
                                        int32_t classes_used, void *h_values);
/* Split forms for callers that allocate their outputs while the device works:
 * _begin uploads the inputs and enqueues the device path into the plan's
 * staging, then returns; _end writes the outputs (same buffer conventions as
 * the _classes / flat forms above) and waits.  One split call per plan at a
 * time (a second _begin, or an _end without its _begin, is
 * MGRG_INVALID_ARGUMENT); no other call may use the plan in between. */
mgrg_status mgrg_decompose_host_begin(mgrg_plan *plan, const void *h_values);
mgrg_status mgrg_decompose_host_end(mgrg_plan *plan, void *const *h_classes);
mgrg_status mgrg_recompose_host_begin(mgrg_plan *plan, const void *const *h_classes,
                                      int32_t classes_used);
mgrg_status mgrg_recompose_host_end(mgrg_plan *plan, void *h_values);
/* Abandon a split call between _begin and _end (waits for its device work). */
mgrg_status mgrg_host_abort(mgrg_plan *plan);

/* ---- unit-level kernels (kernels.hpp), device buffers, for parity ---------
 * compute_coefficients / restore_coefficients (kernels.hpp:284-310): in place
 * on a packed level-`level` array. */
mgrg_status mgrg_gpk(mgrg_plan *plan, int32_t level, int32_t inverse,
                     void *d_level_values, void *stream);
/* masstrans_apply (kernels.hpp:328-412): input extents
 * masstrans_input_shape(level, dim) (kernels.hpp:314-320), output the same
 * with `dim` reduced; fused_copy (dim 0 only, else MGRG_INVALID_FUSION) also
 * writes the level's class (class order) into d_coef. */
mgrg_status mgrg_masstrans(mgrg_plan *plan, int32_t level, int32_t dim,
                           const void *d_in, void *d_out, int32_t fused_copy,
                           void *d_coef, void *stream);
/* solve_correction (kernels.hpp:417-448): in place on the level-(l-1)
 * lattice; identity when `dim` does not refine. */
mgrg_status mgrg_solve(mgrg_plan *plan, int32_t level, int32_t dim, void *d_f,
                       void *stream);
/* apply_correction (kernels.hpp:451-464): values += sign * z. */
mgrg_status mgrg_apply_correction(mgrg_plan *plan, uint64_t count,
                                  void *d_values, const void *d_z, int32_t sign,
                                  void *stream);
/* reorder (grid.hpp:177-196) of one packed level-`level` array: direction 0 =
 * to_hierarchical (coarse nodes first, then class order), 1 = to_natural. */
mgrg_status mgrg_reorder(mgrg_plan *plan, int32_t level, int32_t direction,
                         const void *d_in, void *d_out, void *stream);

/* ---- cooperative multi-GPU decompose ----------------
 * cooperative_decompose (parallel.hpp:227-230, parallel_impl.hpp:691-808):
 * every worker (one GPU, one plan for the WHOLE grid) owns a z slab of the
 * level lattices and runs these steps in lockstep with its neighbours; the
 * host (paper_2105_12764_b200/coop.py) moves the halo planes and the Thomas
 * carries between GPUs (NCCL send/recv or peer copies).  Results are
 * bit-identical to mgrg_decompose of the whole grid (exact policy).
 *
 * mgrg_coop_level: level `level` (3-D, odd extents, z refining) on coarse
 * planes [c0, c1): coefficients, class-`level` stores of fine planes
 * [2c0, 2c1), packed coarse values, the load vector, and its x and y
 * solves.  Reads fine planes [2c0-2, 2c1] of the level array: d_level is the
 * caller's finest-level buffer at level L, NULL below (the plan's level
 * buffer, see mgrg_plan_level_buffer).  c0 (and c1 unless it is the last
 * coarse plane + 1) must be even multiples of a power of two >= 1.
 * mgrg_coop_thomas_z: the z solve of coarse planes [c0, c1) for xy fibers
 * [f0, f1): direction 0 = forward elimination (carry_in = the previous
 * worker's last forward plane, NULL when c0 == 0; carry_out = this worker's
 * last forward plane); direction 1 = back substitution fused with apply_pack
 * (carry_in = the next worker's first solved plane, NULL at the top; carry_out
 * = this worker's first solved plane).  Carries are full xy planes (m0*m1
 * elements) indexed by fiber. */
mgrg_status mgrg_coop_level(mgrg_plan *plan, int32_t level, uint32_t c0, uint32_t c1,
                            const void *d_level, void *d_classes, void *stream);
mgrg_status mgrg_coop_thomas_z(mgrg_plan *plan, int32_t level, uint32_t c0, uint32_t c1,
                               uint64_t f0, uint64_t f1, int32_t direction,
                               const void *d_carry_in, void *d_carry_out, void *d_classes,
                               void *stream);
/* Device pointer of the plan's packed level-`level` buffer (1 <= level < L). */
mgrg_status mgrg_plan_level_buffer(mgrg_plan *plan, int32_t level, void **d_ptr);

/* Fault hook of cooperative runs (CoopOptions::fault_injector,
 * parallel.hpp:68-70): called at every phase entry ("level", "solve",
 * "tail", "serial"); a non-zero return aborts the run as WORKER_FAILURE. */
typedef int (*mgrg_fault_fn)(void *ctx, int32_t worker, const char *phase, int32_t level);
/* cooperative_decompose (parallel_impl.hpp:691-808) of a host grid by
 * `workers` workers, worker w on device (desc->device + w) mod the visible
 * devices (several workers may share a GPU), driven from the calling thread
 * with the steps above; classes (N elements, class l at N_{l-1}) written to
 * h_classes, bit-identical to mgrg_decompose_host of the whole grid (exact
 * policy).  remote_elements (optional) = elements moved between distinct
 * workers (CommReport).  TOO_MANY_WORKERS as make_partitions
 * (parallel.cpp:41-55). */
mgrg_status mgrg_cooperative_decompose_host(const mgrg_grid_desc *desc, int32_t workers,
                                            const void *h_values, void *h_classes,
                                            mgrg_fault_fn fault, void *fault_ctx,
                                            uint64_t *remote_elements);

/* ---- diagnostics ------------------------------------------------------- */
/* Thread-local message of the last failing call ("" if none). */
const char *mgrg_last_error(void);
/* Status name as the reference spells the exception ("InvalidGrid", ...). */
const char *mgrg_status_name(mgrg_status status);
/* CUDA-graph replay (enable != 0): mgrg_decompose / mgrg_recompose capture
 * their level loop (the ~L*5 dependent launches) once per (operation, buffer
 * pointers, classes_used) into a graph on a plan-owned stream and replay it,
 * ordered after and before the caller's stream by events; at most 8 graphs
 * are kept per plan.  Values are identical with and without graphs.  With
 * per-launch profiling on, the profiling events are captured into the graph:
 * the records then hold the launches of the capturing call, timed by the
 * LAST replay. */
mgrg_status mgrg_plan_set_graphs(mgrg_plan *plan, int32_t enable);
/* Kernel launches the last decompose/recompose issued on this plan. */
mgrg_status mgrg_plan_last_launches(const mgrg_plan *plan, uint64_t *launches);
/* Per-launch device timing.  With profiling on, every kernel the plan
 * launches is bracketed by CUDA events on its stream (records accumulate
 * across calls until reset).  mgrg_plan_profile_read waits for the recorded
 * work, then fills up to `cap` entries: kernel kind (mgrg_kernel_kind),
 * level, device milliseconds and the algorithmic HBM bytes of that launch
 * (SURVEY.md §8(d) accounting); *count receives the number recorded.
 * enable > 0 profiles every launch; enable < 0 only the launches of the top
 * -enable levels (L, L-1, ...), keeping the event overhead out of a timed
 * loop's small levels; 0 turns profiling off. */
typedef enum mgrg_kernel_kind {
  MGRG_K_DEC_LEVEL = 0, /* GPK + class store + R*M (decompose)      */
  MGRG_K_THOMAS_X = 1,  /* Thomas along dim 0 (+1, +2: dims 1, 2)   */
  MGRG_K_THOMAS_Y = 2,
  MGRG_K_THOMAS_Z = 3,
  MGRG_K_REC_LOAD = 4,  /* class gather + R*M (recompose)           */
  MGRG_K_REC_GPK = 5    /* coarse + class -> level array (recompose) */
} mgrg_kernel_kind;
mgrg_status mgrg_plan_set_profiling(mgrg_plan *plan, int32_t enable);
mgrg_status mgrg_plan_profile_reset(mgrg_plan *plan);
mgrg_status mgrg_plan_profile_read(mgrg_plan *plan, uint64_t cap, int32_t *kinds,
                                   int32_t *levels, float *ms, uint64_t *bytes,
                                   uint64_t *count);

/* Library version string. */
const char *mgrg_version(void);

/* ---- MGRF container --------------------------------
 * CRC-32 of device bytes (mgr::crc32, pipeline.cpp:13-28: reflected
 * 0xEDB88320, init / final xor 0xFFFFFFFF -- zlib's crc32), computed on the
 * GPU; synchronous on `stream`. */
mgrg_status mgrg_crc32(const void *d_bytes, uint64_t nbytes, uint32_t *crc, void *stream);
/* Per-class CRC-32 of a device class buffer, classes 0..upto -> crcs[0..upto]
 * (the MGRF class records, pipeline.cpp:188-191). */
mgrg_status mgrg_class_crc32(mgrg_plan *plan, const void *d_classes, int32_t upto,
                             uint32_t *crcs, void *stream);
/* mgr::write_refactored (pipeline.cpp:180-206, layout pipeline.hpp:27-39)
 * straight from the device class buffer: byte-identical file; CRCs on the
 * GPU, payload streamed through pinned chunks.  IoError on file failures. */
mgrg_status mgrg_write_refactored(mgrg_plan *plan, const void *d_classes, const char *path,
                                  uint64_t *bytes_written);
/* mgr::read_refactored (pipeline.cpp:233-300) into a device class buffer:
 * classes 0..classes (classes < 0: all) are read -- bytes past that prefix
 * are never touched -- and CRC-checked on the GPU (MGRG_CORRUPT_FILE "crc
 * mismatch in class c"; a short payload gives MGRG_MISSING_CLASS).  The
 * container must describe this plan's grid, dtype and depth. */
mgrg_status mgrg_read_refactored(mgrg_plan *plan, const char *path, int32_t classes,
                                 void *d_classes, int32_t *classes_loaded,
                                 uint64_t *bytes_consumed);

/* ---- compression pipeline ------------------------
 * mgr::compress (pipeline.hpp:149-183) of a device field: decompose, the
 * error-bound search (uniform quantizer starting at 2*eb/(L+1), halved until
 * the full recompose meets eb; at most 25 attempts) and the zigzag-varint
 * coding on the GPU, codec 0 (store) / 1 (zlib) on the host.  *out is a
 * malloc'd "MGRC" container (free with mgrg_free); bytes equal the
 * reference's under the exact arithmetic policy.  MGRG_INVALID_BOUND for
 * eb <= 0, an unknown codec or a bound the quantizer cannot reach. */
mgrg_status mgrg_compress(mgrg_plan *plan, const void *d_values, double error_bound,
                          int32_t codec, uint8_t **out, uint64_t *out_size, double *bin,
                          double *measured);
void mgrg_free(void *ptr);
/* mgr::decompress (pipeline.cpp:517-547) into a device field: container
 * parse + codec on the host, varint decode / dequantize / recompose on the
 * GPU; MGRG_CORRUPT_FILE with the reference's messages. */
mgrg_status mgrg_decompress(mgrg_plan *plan, const uint8_t *bytes, uint64_t size,
                            void *d_values, double *error_bound, double *bin,
                            double *measured, int32_t *codec);

/* Host-buffer forms of the container / compression entry points (the
 * reference's pipeline callers hold host vectors; include/mgr_b200/pipeline.hpp
 * uses these).  Same semantics; staged through the plan's device buffers. */
mgrg_status mgrg_crc32_host(const void *h_bytes, uint64_t nbytes, uint32_t *crc);
mgrg_status mgrg_write_refactored_host(mgrg_plan *plan, const void *h_classes,
                                       const char *path, uint64_t *bytes_written);
mgrg_status mgrg_read_refactored_host(mgrg_plan *plan, const char *path, int32_t classes,
                                      void *h_classes, int32_t *classes_loaded,
                                      uint64_t *bytes_consumed);
mgrg_status mgrg_compress_host(mgrg_plan *plan, const void *h_values, double error_bound,
                               int32_t codec, uint8_t **out, uint64_t *out_size, double *bin,
                               double *measured);
mgrg_status mgrg_decompress_host(mgrg_plan *plan, const uint8_t *bytes, uint64_t size,
                                 void *h_values, double *error_bound, double *bin,
                                 double *measured, int32_t *codec);

/* ---- devices, cooperative schedule ---------------------------------------
 * Visible CUDA devices (embarrassing_decompose's worker -> GPU map,
 * parallel_impl.hpp:810-847: one host thread per GPU). */
mgrg_status mgrg_device_count(int32_t *count);
/* The slab schedule mgrg_cooperative_decompose_host uses for this plan's grid
 * and `workers` workers: *q = number of cooperative (top) levels (0: worker 0
 * runs the whole decompose), bounds[0..workers] = finest-plane z slab
 * boundaries (bounds has workers + 1 entries; untouched when *q == 0).  The
 * C++ drop-in derives CommReport::idle (parallel.cpp:217-258) from it. */
mgrg_status mgrg_coop_schedule(const mgrg_plan *plan, int32_t workers, int32_t *q,
                               uint64_t *bounds);

/* ---- block metadata gather over NCCL --------------------
 * The one collective of the block-sharded path: every rank holds whole
 * blocks (embarrassing_decompose, parallel_impl.hpp:810-847), and a single
 * ncclAllGather of fixed-size per-block records tells every rank where every
 * block's classes are and how large they are (the MGRF class records,
 * pipeline.cpp:180-206, without the payload).  No bulk data crosses GPUs. */
#define MGRG_MAX_CLASSES 32
typedef struct mgrg_block_meta {
  int64_t block_id;                         /* -1: padding record          */
  int32_t rank;                             /* producing rank              */
  int32_t dtype;                            /* 4 | 8                       */
  int32_t ndims;
  int32_t levels;                           /* L; classes 0..L             */
  uint64_t origin[4];                       /* block origin in the field   */
  uint64_t shape[4];
  uint64_t class_bytes[MGRG_MAX_CLASSES];   /* class l byte length         */
  uint32_t class_crc32[MGRG_MAX_CLASSES];   /* mgr::crc32 of class l bytes */
  uint32_t checksum;                        /* crc32 of class_crc32[0..L]  */
  uint32_t reserved;
  double decompose_ms;                      /* device time, caller-supplied */
  double recompose_ms;
} mgrg_block_meta;
/* Fill `meta` for a decomposed block: geometry and class byte lengths from
 * the plan, per-class CRC-32 of d_classes on the GPU (synchronous on
 * `stream`), the checksum of the CRCs; origin (ndims entries, may be NULL =
 * zeros), block id and timings from the caller. */
mgrg_status mgrg_block_meta_fill(mgrg_plan *plan, const void *d_classes, int64_t block_id,
                                 int32_t rank, const uint64_t *origin, double decompose_ms,
                                 double recompose_ms, mgrg_block_meta *meta, void *stream);
/* One communicator per rank, one rank per GPU (NCCL over NVLink/NVSwitch).
 * Rank 0 makes the unique id; the caller ships its 128 bytes to the other
 * ranks (MPI, a TCP store, a file) before every rank calls mgrg_comm_init. */
typedef struct mgrg_comm mgrg_comm;
#define MGRG_COMM_ID_BYTES 128
mgrg_status mgrg_comm_unique_id(uint8_t id[MGRG_COMM_ID_BYTES]);
mgrg_status mgrg_comm_init(const uint8_t id[MGRG_COMM_ID_BYTES], int32_t nranks,
                           int32_t rank, int32_t device, mgrg_comm **comm);
mgrg_status mgrg_comm_destroy(mgrg_comm *comm);
mgrg_status mgrg_comm_size(const mgrg_comm *comm, int32_t *nranks, int32_t *rank);
/* All-gather of `per_rank` records from every rank (pad with block_id = -1
 * when ranks hold different block counts): all[r * per_rank + i] = rank r's
 * mine[i].  Host buffers in and out; one ncclAllGather on the comm's device,
 * ordered after `stream` (may be NULL) and synchronous.  MGRG_NCCL_ERROR on
 * a collective failure. */
mgrg_status mgrg_comm_allgather_block_meta(mgrg_comm *comm, const mgrg_block_meta *mine,
                                           int32_t per_rank, mgrg_block_meta *all,
                                           void *stream);

#ifdef __cplusplus
}
#endif

#endif /* MGRG_H */
