#!/usr/bin/env python3
"""Exact-policy bit-identity of several libmgrg builds on the failing shapes
(plain ctypes: only plan_create / decompose / plan_destroy, so older builds
load)."""
import ctypes
import glob
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402


class GridDesc(ctypes.Structure):
    _fields_ = [("ndims", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("shape", ctypes.c_uint64 * 4), ("coords", ctypes.c_void_p),
                ("levels", ctypes.c_int32), ("device", ctypes.c_int32),
                ("flags", ctypes.c_int32)]


def run(libpath, cases):
    import torch

    lib = ctypes.CDLL(libpath)
    lib.mgrg_plan_create.argtypes = [ctypes.POINTER(GridDesc), ctypes.POINTER(ctypes.c_void_p)]
    lib.mgrg_decompose.argtypes = [ctypes.c_void_p] * 4
    lib.mgrg_plan_destroy.argtypes = [ctypes.c_void_p]
    res = []
    for shape, dt, nonuni, seed in cases:
        rng = np.random.default_rng(seed)
        coords = ([np.cumsum(rng.uniform(0.1, 1.0, n)) for n in shape] if nonuni else None)
        v = rng.random(int(np.prod(shape))).astype(dt)
        d = GridDesc()
        d.ndims = len(shape)
        d.dtype = 4 if dt == "float32" else 8
        for i, n in enumerate(shape):
            d.shape[i] = n
        cf = np.concatenate(coords).astype(np.float64) if coords else None
        d.coords = cf.ctypes.data if cf is not None else None
        d.levels, d.device, d.flags = 0, 0, 0
        h = ctypes.c_void_p()
        assert lib.mgrg_plan_create(ctypes.byref(d), ctypes.byref(h)) == 0
        tv = torch.from_numpy(v).cuda()
        tc = torch.empty_like(tv)
        st = lib.mgrg_decompose(h, ctypes.c_void_p(tv.data_ptr()), ctypes.c_void_p(tc.data_ptr()), None)
        torch.cuda.synchronize()
        ref, _ = oracle.decompose(v, shape, coords)
        res.append((shape, nonuni, seed, st, bool(np.array_equal(tc.cpu().numpy(), ref))))
        lib.mgrg_plan_destroy(h)
    return res


if __name__ == "__main__":
    cases = [((99, 37), "float32", True, 0), ((64, 37), "float32", True, 0),
             ((100, 36), "float32", False, 0), ((100, 9, 5), "float32", True, 0),
             ((12, 10), "float32", True, 0), ((200, 150), "float32", True, 0)]
    libs = sys.argv[1:] or sorted(glob.glob(os.path.join(ROOT, "paper_2105_12764_b200", "variants", "*.so")))
    for lp in libs:
        print(os.path.basename(lp), run(lp, cases), flush=True)
