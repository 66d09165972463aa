"""Unit-level kernels (kernels.hpp:284-464 and grid.hpp:177-196 API: gpk,
masstrans, solve, reorder) through the C ABI against the CPU oracle, bit
for bit, on every level of 3-D and 4-D grids; and decompose_spatiotemporal
(refactor.hpp:536-567) against fixtures written by the reference itself."""
import os
import sys
import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

SHAPES = [(9, 9, 9), (17, 9, 5), (12, 10, 9), (9, 5, 3, 6), (5, 5, 5, 5), (6, 7, 9, 10),
          (17, 9, 5, 3)]


def _setup(shape, dtype, nonuni):
    from paper_2105_12764_b200 import Plan

    rng = np.random.default_rng(zlib.crc32(repr((shape, dtype, nonuni)).encode()))
    coords = [np.cumsum(rng.uniform(0.1, 1.0, n)) for n in shape] if nonuni else None
    return rng, coords, Plan(shape, dtype, coords=coords)


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("nonuni", [False, True], ids=["uniform", "nonuniform"])
def test_unit_kernels_bit_exact(shape, dtype, nonuni, oracle_mod):
    import torch

    rng, coords, plan = _setup(shape, dtype, nonuni)
    L = plan.levels
    nd = len(shape)
    for l in range(1, L + 1):
        ls = tuple(int(x) for x in plan.level_shape(l))
        cs = tuple(int(x) for x in plan.level_shape(l - 1))
        F, C = int(np.prod(ls)), int(np.prod(cs))
        v = rng.standard_normal(F).astype(dtype)
        # gpk forward / inverse on the level-l lattice (kernels.hpp:284-310)
        for inv in (False, True):
            d = torch.from_numpy(v.copy()).cuda()
            plan.gpk(l, d, inverse=inv)
            ref = oracle_mod.gpk(v, shape, l, inv, coords=coords)
            assert np.array_equal(d.cpu().numpy(), ref), f"gpk l={l} inv={inv}"
        # masstrans along each dim (kernels.hpp:328-412), fused copy on dim 0
        for dim in range(nd):
            ie = [cs[k] if k < dim else ls[k] for k in range(nd)]
            oe = list(ie)
            oe[dim] = cs[dim]
            x = rng.standard_normal(int(np.prod(ie))).astype(dtype)
            fused = dim == 0
            ref_o, ref_c = oracle_mod.masstrans(x, shape, l, dim, int(np.prod(oe)),
                                                fused_copy=fused, class_size=F - C,
                                                coords=coords)
            d_out = torch.empty(int(np.prod(oe)), dtype=getattr(torch, dtype), device="cuda")
            d_coef = (torch.zeros(F - C, dtype=getattr(torch, dtype), device="cuda")
                      if fused else None)
            plan.masstrans(l, dim, torch.from_numpy(x).cuda(), d_out, fused_copy=fused,
                           coef=d_coef)
            assert np.array_equal(d_out.cpu().numpy(), ref_o), f"masstrans l={l} dim={dim}"
            if fused:
                assert np.array_equal(d_coef.cpu().numpy(), ref_c), f"class copy l={l}"
        # Thomas along each dim of the level-(l-1) lattice (kernels.hpp:417-448)
        for dim in range(nd):
            f = rng.standard_normal(C).astype(dtype)
            ref = oracle_mod.solve(f, shape, l, dim, coords=coords)
            d = torch.from_numpy(f.copy()).cuda()
            plan.solve(l, dim, d)
            assert np.array_equal(d.cpu().numpy(), ref), f"solve l={l} dim={dim}"
        # coarse-first reorder and its inverse (grid.hpp:177-196)
        ref = oracle_mod.reorder(v.astype(np.float64), shape, l, coords=coords).astype(dtype)
        d_out = torch.empty_like(torch.from_numpy(v)).cuda()
        plan.reorder(l, torch.from_numpy(v).cuda(), d_out)
        assert np.array_equal(d_out.cpu().numpy(), ref), f"reorder l={l}"
        back = torch.empty_like(d_out)
        plan.reorder(l, d_out, back, to_natural=True)
        assert np.array_equal(back.cpu().numpy(), v), f"to_natural l={l}"
    plan.close()


# ---- decompose_spatiotemporal vs the reference -----------------------------
def _st_cases():
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                             "refactor_golden.npz"))
    out = []
    for i in range(int(z["nst"][0])):
        shape = tuple(int(s) for s in z[f"st{i}_shape"])
        coords = None
        if f"st{i}_coords" in z.files:
            flat = z[f"st{i}_coords"]
            coords, o = [], 0
            for n in shape:
                coords.append(flat[o:o + n])
                o += n
        for dt in ("float64", "float32"):
            out.append(dict(id=f"{'x'.join(map(str, shape))}x{len(z[f'st{i}_time'])}-{dt}",
                            shape=shape, coords=coords, time=z[f"st{i}_time"],
                            values=z[f"st{i}_{dt}_values"], classes=z[f"st{i}_{dt}_classes"],
                            levels=int(z[f"st{i}_{dt}_levels"][0])))
    return out


@pytest.mark.parametrize("case", _st_cases(), ids=lambda c: c["id"])
def test_spatiotemporal_matches_reference(case):
    from paper_2105_12764_b200 import decompose_spatiotemporal, make_grid, recompose

    shape, T = case["shape"], len(case["time"])
    n = int(np.prod(shape))
    snaps = [make_grid(shape, case["values"][t * n:(t + 1) * n], case["coords"], 2)
             for t in range(T)]
    r = decompose_spatiotemporal(snaps, case["time"])
    assert r.levels == case["levels"]
    got = np.concatenate([np.asarray(c).reshape(-1) for c in r.classes])
    assert np.array_equal(got, case["classes"])
    back = recompose(r, r.levels)
    err = np.abs(np.asarray(back.values).reshape(-1) - case["values"]).max()
    tol = 1e-4 if case["values"].dtype == np.float32 else 1e-12
    assert err <= tol * (np.ptp(case["values"]) or 1.0)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("n", [1, 255, 256, 257, 100003])
def test_apply_correction_matches_reference(dtype, n):
    """apply_correction (kernels.hpp:451-464): values += z for sign >= 0,
    values -= z otherwise, one IEEE add / subtract per node (numpy's are the
    same round-to-nearest operations); length mismatch is ShapeError."""
    import torch

    from paper_2105_12764_b200 import Plan
    from paper_2105_12764_b200.errors import ShapeError

    rng = np.random.default_rng(n)
    plan = Plan((9, 9), dtype)
    v = rng.standard_normal(n).astype(dtype)
    z = rng.standard_normal(n).astype(dtype)
    for sign, ref in ((1, v + z), (0, v + z), (-1, v - z), (-7, v - z)):
        d = torch.from_numpy(v.copy()).cuda()
        plan.apply_correction(d, torch.from_numpy(z).cuda(), sign)
        assert np.array_equal(d.cpu().numpy(), ref), sign
    with pytest.raises(ShapeError, match="does not match"):
        plan.apply_correction(torch.from_numpy(v).cuda(), torch.from_numpy(z[:-1].copy()).cuda()
                              if n > 1 else torch.zeros(2, dtype=getattr(torch, dtype)).cuda())
    plan.close()
