"""Device-level handle over the C ABI: one plan per (grid geometry, dtype,
device).  Buffers are torch CUDA tensors (device entry points) or numpy
arrays (host entry points); torch is only the allocator/stream provider."""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib, errors

_DTYPES = {"float32": _lib.MGRG_F32, "float64": _lib.MGRG_F64}


def _dtype_name(dtype) -> str:
    s = str(dtype).replace("torch.", "")
    if s in ("float32", "float", "f4", "<f4"):
        return "float32"
    if s in ("float64", "double", "f8", "<f8"):
        return "float64"
    raise errors.InvalidArgument(f"unsupported dtype {dtype}")


def _stream_ptr(stream, device=None):
    """The stream to launch on: torch's current stream OF THE PLAN'S DEVICE
    when none is given (not the current device's)."""
    if stream is None:
        import torch

        return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _tensor_ptr(t):
    if not t.is_cuda:
        raise errors.InvalidArgument("device entry points take CUDA tensors")
    if not t.is_contiguous():
        raise errors.InvalidArgument("tensor must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


class Plan:
    """mgrg_plan: hierarchy + geometry + device workspace for one grid."""

    def __init__(self, shape, dtype="float32", coords=None, levels=None, device=0,
                 fast: bool = False):
        L = _lib.lib()
        self.shape = tuple(int(s) for s in shape)
        self.dtype = _dtype_name(dtype)
        self.np_dtype = np.dtype(self.dtype)
        self.device = int(device)
        desc = _lib.GridDesc()
        desc.ndims = len(self.shape)
        desc.dtype = _DTYPES[self.dtype]
        for d, s in enumerate(self.shape[:4]):
            desc.shape[d] = s
        self._coords = None
        if coords is not None:
            if len(coords) != len(self.shape):
                raise errors.InvalidGrid("coordinate arrays do not match dimension count")
            for d, c in enumerate(coords):
                if len(c) != self.shape[d]:
                    raise errors.InvalidGrid(
                        f"coordinates of dimension {d} do not match its extent")
            self._coords = np.ascontiguousarray(
                np.concatenate([np.asarray(c, dtype=np.float64) for c in coords]))
            desc.coords = self._coords.ctypes.data
        desc.levels = 0 if levels is None else min(int(levels), 64)
        if levels is not None and int(levels) < 1:
            raise errors.InvalidLevel("level count must be at least 1")
        desc.device = self.device
        desc.flags = _lib.MGRG_FLAG_FAST if fast else 0
        self.fast = bool(fast)
        h = ctypes.c_void_p()
        _lib.check(L.mgrg_plan_create(ctypes.byref(desc), ctypes.byref(h)))
        self._h = h
        lv = ctypes.c_int32()
        _lib.check(L.mgrg_plan_levels(h, ctypes.byref(lv)))
        self.levels = lv.value
        off = (ctypes.c_uint64 * (self.levels + 2))()
        _lib.check(L.mgrg_plan_class_offsets(h, off))
        self.class_offsets = [int(x) for x in off]
        n, wsb = ctypes.c_uint64(), ctypes.c_uint64()
        _lib.check(L.mgrg_plan_sizes(h, ctypes.byref(n), ctypes.byref(wsb)))
        self.num_elements = n.value
        self.workspace_bytes = wsb.value

    # -- lifetime -------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().mgrg_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- geometry ---------------------------------------------------------------
    def level_shape(self, level: int):
        ext = (ctypes.c_uint64 * len(self.shape))()
        _lib.check(_lib.lib().mgrg_plan_level_shape(self._h, level, ext))
        return tuple(int(e) for e in ext)

    def class_slices(self):
        o = self.class_offsets
        return [slice(o[l], o[l + 1]) for l in range(self.levels + 1)]

    @property
    def last_launches(self) -> int:
        n = ctypes.c_uint64()
        _lib.check(_lib.lib().mgrg_plan_last_launches(self._h, ctypes.byref(n)))
        return n.value

    # -- per-launch profiling ------------------------------------------------------
    def set_graphs(self, enable=True):
        """Replay decompose / recompose as captured CUDA graphs (one per
        buffers + classes_used; mgrg_plan_set_graphs)."""
        _lib.check(_lib.lib().mgrg_plan_set_graphs(self._h, int(bool(enable))))

    def set_profiling(self, enable=True, top_levels=None):
        """Per-launch CUDA-event timing; top_levels=k profiles only the
        launches of levels L .. L-k+1."""
        mode = 0 if not enable else (-int(top_levels) if top_levels else 1)
        _lib.check(_lib.lib().mgrg_plan_set_profiling(self._h, mode))
        _lib.check(_lib.lib().mgrg_plan_profile_reset(self._h))

    def profile(self, reset: bool = True):
        """[(kernel, level, ms, algorithmic_bytes)] of the launches recorded
        since profiling was enabled / last reset (waits for them)."""
        L = _lib.lib()
        cnt = ctypes.c_uint64()
        _lib.check(L.mgrg_plan_profile_read(self._h, 0, None, None, None, None,
                                            ctypes.byref(cnt)))
        n = cnt.value
        kinds = np.empty(n, np.int32)
        levels = np.empty(n, np.int32)
        ms = np.empty(n, np.float32)
        by = np.empty(n, np.uint64)
        if n:
            _lib.check(L.mgrg_plan_profile_read(self._h, n, kinds.ctypes.data,
                                                levels.ctypes.data, ms.ctypes.data,
                                                by.ctypes.data, ctypes.byref(cnt)))
        if reset:
            _lib.check(L.mgrg_plan_profile_reset(self._h))
        return [(_lib.KERNEL_KINDS[int(k)], int(l), float(t), int(b))
                for k, l, t, b in zip(kinds, levels, ms, by)]

    # -- device entry points (torch CUDA tensors) --------------------------------
    def _torch_dtype(self):
        import torch

        return torch.float32 if self.dtype == "float32" else torch.float64

    def _check_tensor(self, t, n, what):
        if t.dtype != self._torch_dtype():
            raise errors.InvalidArgument(f"{what} has dtype {t.dtype}, plan is {self.dtype}")
        if t.numel() < n:
            raise errors.ShapeError(f"{what} has {t.numel()} elements, need {n}")
        if not t.is_cuda or t.device.index != self.device:
            raise errors.InvalidArgument(
                f"{what} is on {t.device}, plan is on cuda:{self.device}")
        if not t.is_contiguous():
            raise errors.InvalidArgument(f"{what} must be contiguous")

    def decompose(self, values, classes=None, stream=None):
        """mgr::decompose on device buffers; returns the flat class tensor."""
        import torch

        self._check_tensor(values, self.num_elements, "values")
        if classes is None:
            classes = torch.empty(self.num_elements, dtype=values.dtype, device=values.device)
        self._check_tensor(classes, self.num_elements, "classes")
        _lib.check(_lib.lib().mgrg_decompose(self._h, _tensor_ptr(values),
                                             _tensor_ptr(classes), _stream_ptr(stream, self.device)))
        return classes

    def recompose(self, classes, classes_used=None, out=None, stream=None):
        """mgr::recompose on device buffers (classes above classes_used unread)."""
        import torch

        k = self.levels if classes_used is None else int(classes_used)
        if k < 0 or k > self.levels:
            raise errors.InvalidLevel(
                f"requested {k} classes; container has {self.levels}")
        self._check_tensor(classes, self.class_offsets[k + 1], "classes")
        if out is None:
            out = torch.empty(self.num_elements, dtype=classes.dtype, device=classes.device)
        self._check_tensor(out, self.num_elements, "values")
        _lib.check(_lib.lib().mgrg_recompose(self._h, _tensor_ptr(classes), k,
                                             _tensor_ptr(out), _stream_ptr(stream, self.device)))
        return out

    # -- host entry points (numpy) ----------------------------------------------
    def decompose_host(self, values: np.ndarray, out: np.ndarray | None = None):
        v = np.ascontiguousarray(values, dtype=self.np_dtype)
        if v.size != self.num_elements:
            raise errors.ShapeError(
                f"value count {v.size} does not match grid of {self.num_elements} nodes")
        if out is None:
            out = np.empty(self.num_elements, dtype=self.np_dtype)
        _lib.check(_lib.lib().mgrg_decompose_host(self._h, v.ctypes.data, out.ctypes.data))
        return out

    def recompose_host(self, classes: np.ndarray, classes_used=None,
                       out: np.ndarray | None = None):
        k = self.levels if classes_used is None else int(classes_used)
        c = np.ascontiguousarray(classes, dtype=self.np_dtype)
        if k < 0 or k > self.levels:
            raise errors.InvalidLevel(f"requested {k} classes; container has {self.levels}")
        if c.size < self.class_offsets[k + 1]:
            raise errors.MissingClass(f"class {k} not loaded")
        if out is None:
            out = np.empty(self.num_elements, dtype=self.np_dtype)
        _lib.check(_lib.lib().mgrg_recompose_host(self._h, c.ctypes.data, k, out.ctypes.data))
        return out

    # -- MGRF container straight from / into device class buffers ---------------
    def class_crc32(self, classes, upto=None, stream=None):
        """Per-class CRC-32 (the MGRF class records) of a device class buffer."""
        k = self.levels if upto is None else int(upto)
        self._check_tensor(classes, self.class_offsets[k + 1], "classes")
        out = (ctypes.c_uint32 * (k + 1))()
        _lib.check(_lib.lib().mgrg_class_crc32(self._h, _tensor_ptr(classes), k, out,
                                               _stream_ptr(stream, self.device)))
        return [int(x) for x in out]

    def write_refactored(self, classes, path) -> int:
        """mgr::write_refactored (pipeline.cpp:180-206) from the device class
        buffer; returns the bytes written (header + payloads)."""
        self._check_tensor(classes, self.num_elements, "classes")
        n = ctypes.c_uint64(0)
        _lib.check(_lib.lib().mgrg_write_refactored(self._h, _tensor_ptr(classes),
                                                    os.fsencode(str(path)), ctypes.byref(n)))
        return int(n.value)

    def read_refactored(self, path, classes=None, out=None):
        """mgr::read_refactored (pipeline.cpp:233-300) into a device class
        buffer: (tensor, classes_loaded, bytes_consumed); only the header and
        classes 0..classes are read, each CRC-checked on the GPU."""
        import torch

        if out is None:
            out = torch.zeros(self.num_elements, dtype=getattr(torch, self.dtype),
                              device=torch.device("cuda", self.device))
        self._check_tensor(out, self.num_elements, "classes")
        loaded = ctypes.c_int32(0)
        used = ctypes.c_uint64(0)
        _lib.check(_lib.lib().mgrg_read_refactored(
            self._h, os.fsencode(str(path)), -1 if classes is None else int(classes),
            _tensor_ptr(out), ctypes.byref(loaded), ctypes.byref(used)))
        return out, int(loaded.value), int(used.value)

    # -- compression pipeline (pipeline.hpp:149-198) on device fields ---------
    def compress(self, values, error_bound: float, codec: int = 1):
        """mgr::compress of a device field: (container bytes, bin, measured
        max abs error); codec 0 = store, 1 = zlib."""
        self._check_tensor(values, self.num_elements, "values")
        out = ctypes.c_void_p()
        n = ctypes.c_uint64(0)
        b, m = ctypes.c_double(0), ctypes.c_double(0)
        L = _lib.lib()
        _lib.check(L.mgrg_compress(self._h, _tensor_ptr(values), float(error_bound),
                                   int(codec), ctypes.byref(out), ctypes.byref(n),
                                   ctypes.byref(b), ctypes.byref(m)))
        try:
            data = ctypes.string_at(out.value, n.value)
        finally:
            L.mgrg_free(out)
        return data, b.value, m.value

    def decompress(self, data: bytes, out=None):
        """mgr::decompress into a device field: (tensor, error_bound, bin,
        measured, codec id)."""
        import torch

        if out is None:
            out = torch.empty(self.num_elements, dtype=getattr(torch, self.dtype),
                              device=torch.device("cuda", self.device))
        self._check_tensor(out, self.num_elements, "values")
        buf = ctypes.create_string_buffer(bytes(data), len(data))
        e, b, m = ctypes.c_double(0), ctypes.c_double(0), ctypes.c_double(0)
        c = ctypes.c_int32(0)
        _lib.check(_lib.lib().mgrg_decompress(self._h, buf, len(data), _tensor_ptr(out),
                                              ctypes.byref(e), ctypes.byref(b),
                                              ctypes.byref(m), ctypes.byref(c)))
        return out, e.value, b.value, m.value, int(c.value)

    # -- unit-level kernels (kernels.hpp API), device tensors, in order on the
    #    current stream ------------------------------------------------------------
    def gpk(self, level: int, values, inverse: bool = False, stream=None):
        """compute_coefficients / restore_coefficients in place."""
        _lib.check(_lib.lib().mgrg_gpk(self._h, level, int(inverse), _tensor_ptr(values),
                                       _stream_ptr(stream, self.device)))
        return values

    def masstrans(self, level: int, dim: int, inp, out, fused_copy=False, coef=None,
                  stream=None):
        _lib.check(_lib.lib().mgrg_masstrans(
            self._h, level, dim, _tensor_ptr(inp), _tensor_ptr(out), int(fused_copy),
            _tensor_ptr(coef) if coef is not None else None, _stream_ptr(stream, self.device)))
        return out

    def solve(self, level: int, dim: int, f, stream=None):
        _lib.check(_lib.lib().mgrg_solve(self._h, level, dim, _tensor_ptr(f),
                                         _stream_ptr(stream, self.device)))
        return f

    def apply_correction(self, values, z, sign: int = 1, stream=None):
        if values.numel() != z.numel():
            raise errors.ShapeError(
                f"correction length {z.numel()} does not match {values.numel()} nodes")
        _lib.check(_lib.lib().mgrg_apply_correction(
            self._h, values.numel(), _tensor_ptr(values), _tensor_ptr(z), int(sign),
            _stream_ptr(stream, self.device)))
        return values

    def reorder(self, level: int, values, out, to_natural: bool = False, stream=None):
        _lib.check(_lib.lib().mgrg_reorder(self._h, level, int(to_natural),
                                           _tensor_ptr(values), _tensor_ptr(out),
                                           _stream_ptr(stream, self.device)))
        return out
