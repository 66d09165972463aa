"""CPU oracle for the decompose/recompose path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package, and only as the checker (never as the thing
measured or shipped).  The product (paper_2105_12764_b200) never imports it.

Two CPU implementations behind one numpy interface:

* ``impl="oracle"``: oracle/libmgr_oracle.so, the plain-C restatement
  (mgr_oracle.c / mgr_oracle_engine.inc, each function citing the reference
  file:line it restates);
* ``impl="ref"``: oracle/_ref/libmgr_ref.so, the UNMODIFIED reference
  (/root/reference/proj) compiled from its own sources by oracle/Makefile.
  Present wherever ``make -C oracle`` ran with /root/reference mounted (the
  built .so travels to the GPU box with the repo snapshot).

Parity pinned: tests/test_oracle.py asserts the restatement is bit-identical
to the reference on every case and matches the reference tests' golden
vectors (tests/golden/).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(_HERE, "libmgr_oracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libmgr_ref.so")

_libs: dict[str, ctypes.CDLL] = {}


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: status {code}")
        self.code = code


def build(quiet: bool = True) -> None:
    """Compile the oracle (and oracle/_ref when /root/reference exists)."""
    import subprocess

    subprocess.run(["make", "-C", _HERE, "-s"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def available(impl: str = "oracle") -> bool:
    return os.path.exists(ORACLE_SO if impl == "oracle" else REF_SO)


def _lib(impl: str) -> ctypes.CDLL:
    if impl not in _libs:
        path = ORACLE_SO if impl == "oracle" else REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        _libs[impl] = ctypes.CDLL(path)
    return _libs[impl]


def _prefix(impl: str) -> str:
    return "mgro_" if impl == "oracle" else "mgrref_"


def _sfx(dtype) -> str:
    dt = np.dtype(dtype)
    if dt == np.float64:
        return "f64"
    if dt == np.float32:
        return "f32"
    raise TypeError(f"unsupported dtype {dt}")


def _shape_arr(shape):
    return (ctypes.c_uint64 * len(shape))(*[int(s) for s in shape])


def _coords_arr(shape, coords):
    if coords is None:
        return None, None
    flat = np.ascontiguousarray(np.concatenate([np.asarray(c, dtype=np.float64)
                                                for c in coords]))
    if flat.size != sum(int(s) for s in shape):
        raise OracleError(1, "coordinate arrays do not match the shape")
    return flat, flat.ctypes.data_as(ctypes.c_void_p)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(st: int, what: str) -> None:
    if st != 0:
        raise OracleError(st, what)


def hierarchy(shape, coords=None, levels_cap: int = 0, min_extent: int = 2):
    """(L, extents[L+1][ndims]) of build_hierarchy (grid.cpp:78-112)."""
    lib = _lib("oracle")
    nd = len(shape)
    ext = (ctypes.c_uint64 * (65 * nd))()
    lv = ctypes.c_int()
    keep, cp = _coords_arr(shape, coords)
    lib.mgro_hierarchy.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_int, ctypes.c_int,
                                   ctypes.POINTER(ctypes.c_int), ctypes.c_void_p]
    _check(lib.mgro_hierarchy(nd, _shape_arr(shape), cp, levels_cap, min_extent,
                              ctypes.byref(lv), ext), "hierarchy")
    L = lv.value
    return L, [[int(ext[l * nd + d]) for d in range(nd)] for l in range(L + 1)]


def class_offsets(shape, levels: int):
    """offsets[0..L+1]: class l starts at offsets[l] = N_{l-1}."""
    lib = _lib("oracle")
    off = (ctypes.c_uint64 * (levels + 2))()
    lib.mgro_class_offsets.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                       ctypes.c_void_p]
    _check(lib.mgro_class_offsets(len(shape), _shape_arr(shape), levels, off),
           "class_offsets")
    return [int(x) for x in off]


def class_layout(shape, levels: int, level: int):
    lib = _lib("oracle")
    nd = len(shape)
    base = (ctypes.c_uint64 * (1 << nd))()
    ext = (ctypes.c_uint64 * ((1 << nd) * nd))()
    lib.mgro_class_layout.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    _check(lib.mgro_class_layout(nd, _shape_arr(shape), levels, level, base, ext),
           "class_layout")
    return ([int(b) for b in base],
            [[int(ext[m * nd + d]) for d in range(nd)] for m in range(1 << nd)])


def decompose(values: np.ndarray, shape, coords=None, levels_cap: int = 0,
              impl: str = "oracle"):
    """mgr::decompose (refactor.hpp:462-474).  Returns (classes, L) with all
    classes in one flat array, class l at offset N_{l-1}."""
    lib = _lib(impl)
    values = np.ascontiguousarray(values)
    out = np.empty(values.size, dtype=values.dtype)
    fn = getattr(lib, _prefix(impl) + "decompose_" + _sfx(values.dtype))
    fn.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                   ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]
    keep, cp = _coords_arr(shape, coords)
    lv = ctypes.c_int()
    _check(fn(len(shape), _shape_arr(shape), cp, levels_cap, _ptr(values),
              _ptr(out), ctypes.byref(lv)), "decompose")
    return out, lv.value


def ref_spatiotemporal(values: np.ndarray, shape, time_coords, coords=None):
    """mgr::decompose_spatiotemporal (refactor.hpp:536-567) of the reference
    itself: values snapshot-major (len(time_coords) snapshots of `shape`).
    Returns (classes, L)."""
    lib = _lib("ref")
    values = np.ascontiguousarray(values)
    out = np.empty(values.size, dtype=values.dtype)
    fn = getattr(lib, "mgrref_spatiotemporal_" + _sfx(values.dtype))
    fn.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                   ctypes.POINTER(ctypes.c_int)]
    keep, cp = _coords_arr(shape, coords)
    tc = np.ascontiguousarray(time_coords, dtype=np.float64)
    lv = ctypes.c_int()
    _check(fn(len(shape), _shape_arr(shape), cp, len(tc), _ptr(tc), _ptr(values), _ptr(out),
              ctypes.byref(lv)), "decompose_spatiotemporal")
    return out, lv.value


def recompose(classes: np.ndarray, shape, levels: int, classes_used: int,
              coords=None, impl: str = "oracle") -> np.ndarray:
    """mgr::recompose (refactor.hpp:476-496) from the flat class buffer."""
    lib = _lib(impl)
    classes = np.ascontiguousarray(classes)
    out = np.empty(classes.size, dtype=classes.dtype)
    fn = getattr(lib, _prefix(impl) + "recompose_" + _sfx(classes.dtype))
    fn.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                   ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    keep, cp = _coords_arr(shape, coords)
    _check(fn(len(shape), _shape_arr(shape), cp, levels, _ptr(classes),
              classes_used, _ptr(out)), "recompose")
    return out


def gpk(values: np.ndarray, shape, level: int, inverse: bool = False,
        coords=None, levels_cap: int = 0, impl: str = "oracle") -> np.ndarray:
    """compute_coefficients / restore_coefficients (kernels.hpp:284-310) on a
    packed level array; returns a new array."""
    lib = _lib(impl)
    v = np.array(values, copy=True, order="C")
    fn = getattr(lib, _prefix(impl) + "gpk_" + _sfx(v.dtype))
    fn.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                   ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    keep, cp = _coords_arr(shape, coords)
    _check(fn(len(shape), _shape_arr(shape), cp, levels_cap, level, int(inverse),
              _ptr(v)), "gpk")
    return v


def masstrans(inp: np.ndarray, shape, level: int, dim: int, out_size: int,
              fused_copy: bool = False, class_size: int = 0, coords=None,
              levels_cap: int = 0, impl: str = "oracle"):
    """masstrans_apply (kernels.hpp:328-412); returns (out, coef_out|None)."""
    lib = _lib(impl)
    inp = np.ascontiguousarray(inp)
    out = np.empty(out_size, dtype=inp.dtype)
    coef = np.zeros(class_size, dtype=inp.dtype) if fused_copy else None
    fn = getattr(lib, _prefix(impl) + "masstrans_" + _sfx(inp.dtype))
    fn.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                   ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                   ctypes.c_int, ctypes.c_void_p]
    keep, cp = _coords_arr(shape, coords)
    _check(fn(len(shape), _shape_arr(shape), cp, levels_cap, level, dim, _ptr(inp),
              _ptr(out), int(fused_copy), _ptr(coef) if coef is not None else None),
           "masstrans")
    return out, coef


def solve(f: np.ndarray, shape, level: int, dim: int, coords=None,
          levels_cap: int = 0, impl: str = "oracle") -> np.ndarray:
    """solve_correction (kernels.hpp:417-448) on the level-(l-1) lattice."""
    lib = _lib(impl)
    v = np.array(f, copy=True, order="C")
    fn = getattr(lib, _prefix(impl) + "solve_" + _sfx(v.dtype))
    fn.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                   ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    keep, cp = _coords_arr(shape, coords)
    _check(fn(len(shape), _shape_arr(shape), cp, levels_cap, level, dim, _ptr(v)),
           "solve")
    return v


def reorder(values: np.ndarray, shape, level: int, to_natural: bool = False,
            coords=None, levels_cap: int = 0) -> np.ndarray:
    """reorder (grid.hpp:177-196), f64."""
    lib = _lib("oracle")
    v = np.ascontiguousarray(values, dtype=np.float64)
    out = np.empty_like(v)
    lib.mgro_reorder_f64.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_void_p, ctypes.c_void_p]
    keep, cp = _coords_arr(shape, coords)
    _check(lib.mgro_reorder_f64(len(shape), _shape_arr(shape), cp, levels_cap, level,
                                int(to_natural), _ptr(v), _ptr(out)), "reorder")
    return out


def embarrassing_roundtrip_f32(values: np.ndarray, shape, nblocks: int,
                               workers: int):
    """Reference embarrassing_decompose (parallel_impl.hpp:810-847) + threaded
    recompose of nblocks independent blocks; returns (t_dec, t_rec) seconds."""
    lib = _lib("ref")
    v = np.ascontiguousarray(values, dtype=np.float32)
    fn = lib.mgrref_embarrassing_roundtrip_f32
    fn.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                   ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    td, tr = ctypes.c_double(), ctypes.c_double()
    _check(fn(len(shape), _shape_arr(shape), nblocks, workers, _ptr(v), None, None,
              ctypes.byref(td), ctypes.byref(tr)), "embarrassing_roundtrip")
    return td.value, tr.value


# ---- deterministic data (tests/oracle.cpp:167-186, acceptance.cpp:383-393) --

def smooth_field(shape, coords=None) -> np.ndarray:
    """The reference's smooth test field S(x) evaluated in fp64 on the grid
    (acceptance.cpp:383-393; 2-D drops z, 1-D drops y,z)."""
    axes = []
    for d, n in enumerate(shape):
        axes.append(np.asarray(coords[d], dtype=np.float64) if coords is not None
                    else np.arange(n, dtype=np.float64) / (n - 1))
    c1 = (0.35, 0.4, 0.45)
    c2 = (0.7, 0.65, 0.6)
    # arrays indexed [..., x] with x fastest -> reverse axis order for meshgrid
    grids = np.meshgrid(*axes[::-1], indexing="ij")[::-1]
    r1 = sum((g - c1[d]) ** 2 for d, g in enumerate(grids))
    r2 = sum((g - c2[d]) ** 2 for d, g in enumerate(grids))
    s = np.ones_like(grids[0])
    for g in grids:
        s = s * np.sin(2 * np.pi * g)
    return (np.exp(-30 * r1) + 0.6 * np.exp(-25 * r2) + 0.2 * s).reshape(-1)


def ref_random_vector(n: int, seed: int, lo: float = 0.0, hi: float = 1.0):
    """oracle::random_vector of the reference tests (tests/oracle.cpp:167-174)."""
    lib = _lib("ref")
    out = np.empty(n, dtype=np.float64)
    lib.mgrref_random_vector.argtypes = [ctypes.c_uint64, ctypes.c_uint, ctypes.c_double,
                                         ctypes.c_double, ctypes.c_void_p]
    lib.mgrref_random_vector(n, seed, lo, hi, _ptr(out))
    return out


def ref_random_increasing_coords(n: int, seed: int):
    """oracle::random_increasing_coords (tests/oracle.cpp:176-186)."""
    lib = _lib("ref")
    out = np.empty(n, dtype=np.float64)
    lib.mgrref_random_increasing_coords.argtypes = [ctypes.c_uint64, ctypes.c_uint,
                                                    ctypes.c_void_p]
    lib.mgrref_random_increasing_coords(n, seed, _ptr(out))
    return out


# ---- MGRF container (reference pipeline.cpp:180-300), impl="ref" only -------
def ref_write_refactored(classes, shape, levels, path, coords=None) -> int:
    """The reference's mgr::write_refactored on the RefactoredData given by
    its flat class buffer; returns the bytes written."""
    lib = _lib("ref")
    classes = np.ascontiguousarray(classes)
    fn = getattr(lib, f"mgrref_write_refactored_{_sfx(classes.dtype)}")
    fn.restype = ctypes.c_int64
    keep, cptr = _coords_arr(shape, coords)
    n = fn(ctypes.c_int(len(shape)), _shape_arr(shape), cptr,
           ctypes.c_int(levels), classes.ctypes.data_as(ctypes.c_void_p),
           os.fsencode(path))
    del keep
    if n < 0:
        raise OracleError(int(-n), "mgrref_write_refactored")
    return int(n)


def ref_read_refactored(path, n_elements, dtype, classes=-1):
    """The reference's mgr::read_refactored: (flat classes 0..k, k loaded,
    bytes consumed); raises OracleError(code) like the reference throws."""
    lib = _lib("ref")
    out = np.zeros(n_elements, dtype=dtype)
    loaded = ctypes.c_int(0)
    lib.mgrref_read_refactored.restype = ctypes.c_int64
    n = lib.mgrref_read_refactored(os.fsencode(path), ctypes.c_int(classes),
                                   out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(loaded))
    if n < 0:
        raise OracleError(int(-n), "mgrref_read_refactored")
    return out, loaded.value, int(n)


def ref_crc32(data: bytes) -> int:
    """mgr::crc32 (pipeline.cpp:13-28)."""
    lib = _lib("ref")
    lib.mgrref_crc32.restype = ctypes.c_uint32
    buf = np.frombuffer(bytes(data), dtype=np.uint8)
    return int(lib.mgrref_crc32(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_uint64(buf.size)))


def ref_compress(values, shape, error_bound, codec=1, coords=None):
    """The reference's mgr::compress: (container bytes, bin, measured)."""
    lib = _lib("ref")
    values = np.ascontiguousarray(values)
    fn = getattr(lib, f"mgrref_compress_{_sfx(values.dtype)}")
    fn.restype = ctypes.c_int64
    cap = values.nbytes * 3 + (1 << 20)
    out = np.empty(cap, dtype=np.uint8)
    b, m = ctypes.c_double(0), ctypes.c_double(0)
    keep, cptr = _coords_arr(shape, coords)
    n = fn(ctypes.c_int(len(shape)), _shape_arr(shape), cptr, _ptr(values),
           ctypes.c_double(error_bound), ctypes.c_int(codec), _ptr(out), ctypes.c_uint64(cap),
           ctypes.byref(b), ctypes.byref(m))
    del keep
    if n < 0:
        raise OracleError(int(-n), "mgrref_compress")
    return out[:n].tobytes(), b.value, m.value


def ref_decompress(data: bytes, n_elements, dtype):
    """The reference's mgr::decompress -> flat values."""
    lib = _lib("ref")
    lib.mgrref_decompress.restype = ctypes.c_int64
    buf = np.frombuffer(bytes(data), dtype=np.uint8)
    out = np.zeros(n_elements, dtype=dtype)
    rc = lib.mgrref_decompress(_ptr(buf), ctypes.c_uint64(buf.size), _ptr(out),
                               ctypes.c_uint64(n_elements))
    if rc < 0:
        raise OracleError(int(-rc), "mgrref_decompress")
    return out


def ref_pass_stats(values: np.ndarray, shape, coords=None, levels_cap: int = 0,
                   recompose: bool = False):
    """The reference engine's PassStats (refactor.hpp:223-421) of a decompose
    (+ a full recompose into the same stats when `recompose`): list of
    per-level dicts in the reference's record order."""
    lib = _lib("ref")
    nd = len(shape)
    v = np.ascontiguousarray(values, dtype=np.float64)
    cflat, cptr = _coords_arr(shape, coords)
    w = 8 + 4 * nd
    out = np.zeros(128 * w, dtype=np.uint64)
    n = ctypes.c_int(0)
    fn = lib.mgrref_pass_stats_f64
    fn.restype = ctypes.c_int
    _check(fn(nd, _shape_arr(shape), cptr, int(levels_cap), _ptr(v), int(bool(recompose)),
              _ptr(out), 128, ctypes.byref(n)), "pass_stats")
    recs = []
    for i in range(n.value):
        o = [int(x) for x in out[i * w:(i + 1) * w]]
        recs.append({"level": o[0], "level_elements": o[1], "coefficient": (o[2], o[3]),
                     "fused_copy": (o[4], o[5]),
                     "masstrans": [(o[6 + 2 * d], o[7 + 2 * d]) for d in range(nd)],
                     "solve": [(o[6 + 2 * nd + 2 * d], o[7 + 2 * nd + 2 * d])
                               for d in range(nd)],
                     "apply": (o[6 + 4 * nd], o[7 + 4 * nd])})
    return recs


def embarrassing_roundtrip_blocks_f32(blocks, shape, workers: int, coords=None):
    """Reference embarrassing_decompose + threaded recompose of the given
    same-shape f32 blocks (`blocks`: one C-contiguous array of nblocks * N
    values; `coords`: nblocks * sum(shape) doubles or None); returns
    (t_dec, t_rec) seconds (block copies excluded from the timing)."""
    lib = _lib("ref")
    v = np.ascontiguousarray(blocks, dtype=np.float32)
    n = int(np.prod(shape))
    nblocks = v.size // n
    fn = lib.mgrref_embarrassing_roundtrip_coords_f32
    fn.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                   ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    c = None if coords is None else np.ascontiguousarray(coords, dtype=np.float64)
    td, tr = ctypes.c_double(), ctypes.c_double()
    _check(fn(len(shape), _shape_arr(shape), nblocks, workers,
              None if c is None else _ptr(c), _ptr(v), None, None, ctypes.byref(td),
              ctypes.byref(tr)), "embarrassing_roundtrip")
    return td.value, tr.value
