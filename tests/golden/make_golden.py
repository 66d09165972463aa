#!/usr/bin/env python3
"""Generate the golden fixtures of the decompose/recompose path FROM THE
REFERENCE ITSELF (oracle/_ref/libmgr_ref.so, i.e. /root/reference/proj
compiled from its own sources by oracle/Makefile with the reference's flags).

Run in a container where /root/reference is mounted:
    make -C oracle && python tests/golden/make_golden.py
The output tests/golden/refactor_golden.npz is committed; the parity tests
(CPU oracle and CUDA path) read it and never need /root/reference.

Inputs follow the reference's own test data generators where they exist:
values = oracle::random_vector(N, seed) (tests/oracle.cpp:167-174), non-uniform
coordinates = oracle::random_increasing_coords(n, seed + d)
(tests/oracle.cpp:176-186), as random_grid does (acceptance.cpp:39-50).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (test infrastructure)

# (shape, nonuniform, levels_cap) -- 1-D/2-D/3-D, dyadic and non-dyadic,
# odd and even extents, non-refining extent-2 dims, a depth cap.
CASES = [
    ((5,), False, 0), ((33,), True, 0), ((6,), False, 0), ((12,), True, 0),
    ((65,), False, 0), ((3,), False, 0), ((2, 9), False, 0), ((9, 2), True, 0),
    ((9, 17), True, 0), ((12, 10), False, 0), ((6, 4), True, 0), ((33, 33), False, 0),
    ((65, 40), True, 0), ((33, 33), True, 2),
    ((3, 3, 3), False, 0), ((5, 7, 4), True, 0), ((9, 2, 5), False, 0),
    ((2, 5, 9), True, 0), ((12, 10, 9), False, 0), ((12, 10, 9), True, 0),
    ((17, 9, 5), True, 0), ((17, 17, 17), False, 0), ((17, 17, 17), True, 1),
    ((9, 9, 33), True, 0),
    # 4-D (the stacked grids of decompose_spatiotemporal, refactor.hpp:536-567)
    ((5, 5, 5, 5), False, 0), ((9, 5, 3, 6), True, 0), ((6, 7, 9, 10), True, 0),
    ((17, 9, 5, 3), False, 0), ((9, 9, 9, 9), True, 2), ((5, 3, 2, 9), False, 0),
]

# decompose_spatiotemporal series: (snapshot shape, snapshot count, nonuniform)
ST_CASES = [((9, 5, 5), 5, True), ((17, 9), 3, False), ((5, 5, 5), 2, False)]


def main() -> None:
    if not oracle.available("ref"):
        sys.exit("oracle/_ref/libmgr_ref.so missing: run `make -C oracle` with "
                 "/root/reference mounted")
    arrays = {}
    for i, (shape, nonuni, cap) in enumerate(CASES):
        seed = 1000 + 17 * i
        n = int(np.prod(shape))
        coords = ([oracle.ref_random_increasing_coords(s, seed + d)
                   for d, s in enumerate(shape)] if nonuni else None)
        v64 = oracle.ref_random_vector(n, seed)
        for dt in ("float64", "float32"):
            v = v64.astype(dt)
            cls, L = oracle.decompose(v, shape, coords, cap, impl="ref")
            key = f"c{i}_{dt}"
            arrays[key + "_values"] = v
            arrays[key + "_classes"] = cls
            # progressive reconstructions: every k for small cases, else
            # k = 0, L-1, L
            ks = range(L + 1) if n <= 2000 else sorted({0, max(0, L - 1), L})
            for k in ks:
                arrays[key + f"_rec{k}"] = oracle.recompose(cls, shape, L, k, coords,
                                                            impl="ref")
            arrays[key + "_levels"] = np.array([L])
        arrays[f"c{i}_shape"] = np.array(shape, dtype=np.int64)
        arrays[f"c{i}_cap"] = np.array([cap])
        if coords is not None:
            arrays[f"c{i}_coords"] = np.concatenate(coords)
    # known-answer vectors of the reference tests
    # Fig. 2 (test_refactor.cpp:41-56, test_kernels.cpp:35-46)
    arrays["fig2_values"] = np.array([6.0, 2.0, 0.0, 0.0, 2.0])
    arrays["fig2_coords"] = np.arange(5, dtype=np.float64)
    arrays["fig2_classes"], _ = oracle.decompose(arrays["fig2_values"], (5,),
                                                 [arrays["fig2_coords"]], impl="ref")
    # decompose_spatiotemporal of the reference (values snapshot-major)
    for i, (shape, T, nonuni) in enumerate(ST_CASES):
        seed = 5000 + 31 * i
        n = int(np.prod(shape))
        coords = ([oracle.ref_random_increasing_coords(s, seed + d)
                   for d, s in enumerate(shape)] if nonuni else None)
        tc = oracle.ref_random_increasing_coords(T, seed + 9)
        v64 = oracle.ref_random_vector(n * T, seed)
        for dt in ("float64", "float32"):
            v = v64.astype(dt)
            cls, L = oracle.ref_spatiotemporal(v, shape, tc, coords)
            arrays[f"st{i}_{dt}_values"] = v
            arrays[f"st{i}_{dt}_classes"] = cls
            arrays[f"st{i}_{dt}_levels"] = np.array([L])
        arrays[f"st{i}_shape"] = np.array(shape, dtype=np.int64)
        arrays[f"st{i}_time"] = tc
        if coords is not None:
            arrays[f"st{i}_coords"] = np.concatenate(coords)
    out = os.path.join(HERE, "refactor_golden.npz")
    np.savez_compressed(out, ncases=np.array([len(CASES)]), nst=np.array([len(ST_CASES)]),
                        **arrays)
    print(f"wrote {out}: {len(arrays)} arrays, {os.path.getsize(out)} bytes")


if __name__ == "__main__":
    main()
