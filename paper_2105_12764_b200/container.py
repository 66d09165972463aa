"""MGRF container, mirroring the reference's
include/mgr/pipeline.hpp:15-63 / src/pipeline.cpp:13-300:

* ``crc32(tensor)`` -- mgr::crc32 of device bytes, computed on the GPU;
* ``read_refactored_header(path)`` -- mgr::read_refactored_header (host
  parse, same checks and messages);
* ``write_refactored(r, path)`` / ``read_refactored(path, classes=None)`` --
  the reference's entry points on RefactoredData, running through the device
  path (classes streamed from / into the device class buffer, per-class CRCs
  on the GPU): files are byte-identical to the reference writer's.

Plan.write_refactored / Plan.read_refactored are the device-buffer forms.

Compression pipeline (pipeline.hpp:149-198):
``compress(grid, error_bound, codec="zlib")`` / ``decompress(bytes)`` with the
decompose, the quantizer's error-bound search and the zigzag-varint coding on
the GPU and the codec (store / zlib) on the host; Plan.compress /
Plan.decompress are the device-field forms."""
from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _lib, errors

_MAGIC = b"MGRF"
_VERSION = 1


def crc32(buf) -> int:
    """CRC-32 (zlib's, = mgr::crc32) of a CUDA tensor's bytes, on the GPU."""
    out = ctypes.c_uint32(0)
    nbytes = buf.numel() * buf.element_size()
    _lib.check(_lib.lib().mgrg_crc32(ctypes.c_void_p(buf.data_ptr()), nbytes,
                                     ctypes.byref(out), None))
    return int(out.value)


@dataclass
class ClassRecord:
    bytes: int = 0
    crc: int = 0


@dataclass
class RefactorFileHeader:
    """pipeline.hpp:30-39."""
    version: int = 1
    dtype: int = 8
    shape: tuple = ()
    coords: list = field(default_factory=list)
    levels: int = 0
    class_records: list = field(default_factory=list)
    header_bytes: int = 0

    @property
    def np_dtype(self):
        return np.dtype(np.float32 if self.dtype == 4 else np.float64)


def read_refactored_header(path) -> RefactorFileHeader:
    """mgr::read_refactored_header (pipeline.cpp:220-231, read_header_fields
    :145-177): one bounded read of the file's first MiB."""
    try:
        with open(path, "rb") as f:
            buf = f.read(1 << 20)
    except OSError as e:
        raise errors.IoError(f"cannot open: {path}") from e
    at = 0

    def take(n):
        nonlocal at
        if at + n > len(buf):
            raise errors.CorruptFile("unexpected end of data")
        s = buf[at:at + n]
        at += n
        return s

    if take(4) != _MAGIC:
        raise errors.CorruptFile("bad magic")
    h = RefactorFileHeader()
    h.version = take(1)[0]
    if h.version != _VERSION:
        raise errors.CorruptFile(f"unsupported version {h.version}")
    if take(1)[0] != 0:
        raise errors.CorruptFile("unsupported endianness")
    h.dtype = take(1)[0]
    if h.dtype not in (4, 8):
        raise errors.CorruptFile(f"unsupported dtype {h.dtype}")
    nd = take(1)[0]
    if nd < 1 or nd > 4:
        raise errors.CorruptFile("bad dimension count")
    shape = []
    for _ in range(nd):
        e = struct.unpack("<Q", take(8))[0]
        if e < 2:
            raise errors.CorruptFile("bad dimension size")
        shape.append(e)
    h.shape = tuple(shape)
    h.coords = [np.frombuffer(take(8 * n), dtype="<f8").copy() for n in shape]
    h.levels = struct.unpack("<Q", take(8))[0]
    if h.levels > 64:
        raise errors.CorruptFile("implausible level count")
    for _ in range(h.levels + 1):
        nb, crc = struct.unpack("<QI", take(12))
        h.class_records.append(ClassRecord(nb, crc))
    h.header_bytes = at
    return h


def _plan_for_header(h: RefactorFileHeader, device: int):
    from .refactor import _plan_for, uniform_coords

    uni = all(np.array_equal(c, uniform_coords(n)) for c, n in zip(h.coords, h.shape))
    return _plan_for(h.shape, None if uni else h.coords, h.np_dtype.name, int(h.levels),
                     device)


def write_refactored(r, path, device: int = 0) -> int:
    """mgr::write_refactored (pipeline.cpp:208-215) of a RefactoredData."""
    import torch

    from .refactor import _plan_for, _validate_geometry, flat_if_current, uniform_coords

    _validate_geometry(r.shape, r.coords, 2)
    uni = all(np.array_equal(np.asarray(c, dtype=np.float64), uniform_coords(n))
              for c, n in zip(r.coords, r.shape))
    first = r.classes[0]
    dt = str(first.dtype).replace("torch.", "")
    plan = _plan_for(r.shape, None if uni else r.coords, dt, int(r.levels), device)
    if plan.levels != r.levels:
        raise errors.InvalidLevel(f"container levels {r.levels} do not match the grid")
    if len(r.classes) != plan.levels + 1:
        raise errors.MissingClass(f"write_refactored needs all {plan.levels + 1} classes; "
                                  f"got {len(r.classes)}")
    offs = plan.class_offsets
    for l, c in enumerate(r.classes):
        n = c.numel() if hasattr(c, "is_cuda") else np.asarray(c).size
        if n != offs[l + 1] - offs[l]:
            raise errors.ShapeError(f"class {l} has {n} entries, expected "
                                    f"{offs[l + 1] - offs[l]}")
    flat = flat_if_current(r, plan)
    if flat is None:
        parts = [c.reshape(-1) if hasattr(c, "is_cuda") else
                 torch.from_numpy(np.ascontiguousarray(c).reshape(-1)) for c in r.classes]
        flat = torch.cat([p.to(f"cuda:{device}") for p in parts])
    elif not hasattr(flat, "is_cuda"):
        flat = torch.from_numpy(np.ascontiguousarray(flat)).to(f"cuda:{device}")
    return plan.write_refactored(flat, path)


@dataclass
class ReadResult:
    data: object
    header: RefactorFileHeader
    bytes_consumed: int = 0
    classes_loaded: int = 0


def read_refactored(path, classes=None, device: int = 0) -> ReadResult:
    """mgr::read_refactored (pipeline.cpp:233-300): header plus classes
    0..classes (default all) into a RefactoredData whose classes are views of
    one device buffer; CRC mismatches raise CorruptFile, a short payload
    MissingClass."""
    from .refactor import RefactoredData

    h = read_refactored_header(path)
    want = h.levels if classes is None else int(classes)
    if want > h.levels:
        raise errors.MissingClass(
            f"requested class {want} of a container with {h.levels + 1} classes")
    plan = _plan_for_header(h, device)
    flat, loaded, used = plan.read_refactored(path, want)
    sl = plan.class_slices()[: want + 1]
    data = RefactoredData(tuple(h.shape), [c.copy() for c in h.coords], int(h.levels),
                          [flat[s] for s in sl], None)
    return ReadResult(data, h, used, loaded)


# ---- compression pipeline ----------------------------------------------------
_CODECS = {"store": 0, "zlib": 1}
_CODEC_NAMES = {v: k for k, v in _CODECS.items()}


@dataclass
class CompressionReport:
    """pipeline.hpp:90-96."""
    error_bound: float = 0.0
    bin_width: float = 0.0
    measured_max_abs_error: float = 0.0
    compression_ratio: float = 0.0
    codec: str = ""


@dataclass
class CompressResult:
    bytes: bytes
    report: CompressionReport


@dataclass
class DecompressResult:
    grid: object
    report: CompressionReport


def compress(grid, error_bound: float, codec: str = "zlib", opt=None) -> CompressResult:
    """mgr::compress (pipeline.hpp:149-183) of a TensorGrid."""
    import torch

    from .refactor import RefactorOptions, _all_uniform, _plan_for, _validate_geometry

    opt = opt or RefactorOptions()
    if not error_bound > 0:
        raise errors.InvalidBound("error bound must be positive")
    if codec not in _CODECS:
        raise errors.InvalidBound(f"unknown codec: {codec}")
    _validate_geometry(grid.shape, grid.coords, 2)
    vals = grid.values
    plan = _plan_for(grid.shape, grid.coords if not _all_uniform(grid) else None,
                     vals.dtype, opt.levels, opt.device)
    d = vals.reshape(-1) if hasattr(vals, "is_cuda") else \
        torch.from_numpy(np.ascontiguousarray(vals).reshape(-1)).to(f"cuda:{opt.device}")
    data, b, m = plan.compress(d, error_bound, _CODECS[codec])
    raw = plan.num_elements * np.dtype(plan.dtype).itemsize
    return CompressResult(data, CompressionReport(error_bound, b, m, raw / len(data), codec))


def _compressed_header(data: bytes):
    """parse_compressed_container's header fields (pipeline.cpp:476-503)."""
    at = 0

    def take(n):
        nonlocal at
        if at + n > len(data):
            raise errors.CorruptFile("unexpected end of data")
        s = data[at:at + n]
        at += n
        return s

    if take(4) != b"MGRC":
        raise errors.CorruptFile("bad magic")
    if take(1)[0] != _VERSION:
        raise errors.CorruptFile("unsupported version")
    codec = take(1)[0]
    dt = take(1)[0]
    if dt not in (4, 8):
        raise errors.CorruptFile("unsupported dtype")
    nd = take(1)[0]
    if nd < 1 or nd > 4:
        raise errors.CorruptFile("bad dimension count")
    shape = tuple(struct.unpack("<Q", take(8))[0] for _ in range(nd))
    coords = [np.frombuffer(take(8 * n), dtype="<f8").copy() for n in shape]
    levels = struct.unpack("<Q", take(8))[0]
    if levels > 64:
        raise errors.CorruptFile("implausible level count")
    if codec not in _CODEC_NAMES:
        raise errors.CorruptFile(f"unknown codec id {codec}")
    return codec, dt, shape, coords, levels


def decompress(data: bytes, device: int = 0) -> DecompressResult:
    """mgr::decompress (pipeline.cpp:517-547) -> TensorGrid on the device."""
    from .refactor import TensorGrid, _plan_for, uniform_coords

    codec, dt, shape, coords, levels = _compressed_header(data)
    uni = all(np.array_equal(c, uniform_coords(n)) for c, n in zip(coords, shape))
    plan = _plan_for(shape, None if uni else coords, "float32" if dt == 4 else "float64",
                     int(levels), device)
    out, e, b, m, c = plan.decompress(data)
    grid = TensorGrid(tuple(shape), [c_.copy() for c_ in coords], out)
    raw = plan.num_elements * dt
    return DecompressResult(grid, CompressionReport(e, b, m, raw / len(data), _CODEC_NAMES[c]))
