"""Parity of the CUDA path (through the C ABI) with the CPU oracle.

The device kernels evaluate the reference's expressions in the reference's
order without FMA contraction, so the bar is BIT-EXACT equality with the
oracle (itself pinned bit-exact to the reference in test_oracle.py), on
every class and every progressive reconstruction."""
import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [
    (5,), (33,), (6,), (12,), (65,), (3,), (1025,),
    (9, 17), (33, 5), (12, 10), (6, 4), (2, 9), (9, 2), (65, 65), (129, 67),
    (9, 9, 9), (17, 9, 5), (12, 10, 9), (5, 7, 4), (3, 3, 3), (9, 2, 5), (2, 5, 9),
    (33, 33, 33), (65, 40, 37), (66, 35, 19), (70, 3, 9),
    # multi-tile / multi-chunk pair-lane paths (x tiles of 30, y of 8/16,
    # z chunks of 32 coarse planes), odd and even extents
    (129, 17, 9), (17, 9, 129), (66, 35, 99), (100, 70, 80), (257, 33, 70),
    (61, 62, 64), (200, 150), (4097, 5), (5, 300),
]


def _coords(rng, shape, nonuni):
    if not nonuni:
        return None
    return [np.cumsum(rng.uniform(0.1, 1.0, n)) for n in shape]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("nonuni", [False, True], ids=["uniform", "nonuniform"])
def test_decompose_recompose_bit_exact(shape, dtype, nonuni, oracle_mod):
    import torch

    from paper_2105_12764_b200 import Plan

    rng = np.random.default_rng(zlib.crc32(repr((shape, dtype, nonuni)).encode()))
    coords = _coords(rng, shape, nonuni)
    v = rng.random(int(np.prod(shape))).astype(dtype)
    plan = Plan(shape, dtype, coords=coords)
    ref_c, L = oracle_mod.decompose(v, shape, coords)
    assert plan.levels == L
    d_c = plan.decompose(torch.from_numpy(v).cuda())
    got = d_c.cpu().numpy()
    for l, s in enumerate(plan.class_slices()):
        assert np.array_equal(got[s], ref_c[s]), (
            f"class {l} differs: max |d| = {np.abs(got[s] - ref_c[s]).max()}")
    for k in range(L + 1):
        ref_r = oracle_mod.recompose(ref_c, shape, L, k, coords)
        d_r = plan.recompose(d_c, k)
        assert np.array_equal(d_r.cpu().numpy(), ref_r), f"recompose k={k} differs"
