#!/usr/bin/env python3
"""Golden MGRF containers written by the REFERENCE (mgr::write_refactored,
/root/reference/proj/src/pipeline.cpp:180-206, compiled into oracle/_ref) from
the reference's own decompose of seeded fields.  Run in the build container
(needs /root/reference):  python tests/golden/make_mgrf_golden.py
Writes tests/golden/mgrf/<case>.mgrf and tests/golden/mgrf/cases.npz
(inputs + the reference's classes and bytes_consumed of prefix reads)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

CASES = [  # (name, shape, dtype, nonuniform)
    ("c3d_f64", (17, 9, 5), "float64", False),
    ("c3d_f32_nonuni", (9, 17, 9), "float32", True),
    ("c2d_f32", (33, 17), "float32", False),
    ("c2d_f64_nonuni", (12, 10), "float64", True),
    ("c1d_f64", (65,), "float64", False),
    ("c4d_f32_nonuni", (9, 5, 3, 6), "float32", True),
]


def main():
    out = os.path.join(HERE, "mgrf")
    os.makedirs(out, exist_ok=True)
    arrays = {}
    for i, (name, shape, dt, nonuni) in enumerate(CASES):
        rng = np.random.default_rng(1000 + i)
        coords = ([np.cumsum(rng.uniform(0.1, 1.0, n)) for n in shape] if nonuni else None)
        v = rng.random(int(np.prod(shape))).astype(dt)
        c, L = oracle.decompose(v, shape, coords, impl="ref")
        path = os.path.join(out, f"{name}.mgrf")
        oracle.ref_write_refactored(c, shape, L, path, coords)
        consumed = []
        for k in range(L + 1):
            _, _, used = oracle.ref_read_refactored(path, c.size, dt, k)
            consumed.append(used)
        arrays[f"{name}/values"] = v
        arrays[f"{name}/classes"] = c
        arrays[f"{name}/shape"] = np.array(shape, dtype=np.int64)
        arrays[f"{name}/levels"] = np.array(L)
        arrays[f"{name}/consumed"] = np.array(consumed, dtype=np.int64)
        if coords is not None:
            for d, cd in enumerate(coords):
                arrays[f"{name}/coords{d}"] = np.asarray(cd, dtype=np.float64)
        print(name, shape, dt, "L", L, os.path.getsize(path), "bytes")
    np.savez_compressed(os.path.join(out, "cases.npz"), **arrays)


if __name__ == "__main__":
    main()
