"""Oracle parity at the BASELINE configs' FULL sizes (BASELINE.json configs
1-5) and at the cheap shapes that reach the kernel instantiations the
headline configs use.

A round trip cannot see a wrong correction (a wrong Thomas or mass-transfer
z is added on decompose and subtracted on recompose), so every case here
compares with the CPU oracle directly (oracle/, pinned bit-exact to the
reference in test_oracle.py; its row loops run on all host threads, which
never changes a value):

* decompose: every class of the GPU output against the oracle's classes;
* recompose: the GPU recompose OF THE ORACLE'S CLASSES at k in {0, L/2, L}
  against the oracle's recompose of the same classes (isolates recompose
  from decompose error).

Bars (north_star): exact policy (the C ABI default) =
bit-identical; FAST policy = per class max|gpu - oracle| <= tol * range(input),
tol = 1e-5 (f32) / 1e-12 (f64).  Comparisons run on the device (the arrays
are GBs)."""
import os
import sys
import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

TOL = {"float32": 1e-5, "float64": 1e-12}


def _smooth_field_separable(shape, coords, dtype):
    """The reference's smooth test field (acceptance.cpp:383-393) in fp64 on
    the host, evaluated as the bench does (separable factors), cast to the
    run dtype.  3-D and 2-D."""
    c1, c2 = (0.35, 0.4, 0.45), (0.7, 0.65, 0.6)
    xs = [np.asarray(coords[d], dtype=np.float64) for d in range(len(shape))]
    e1 = [np.exp(-30 * (x - c1[d]) ** 2) for d, x in enumerate(xs)]
    e2 = [np.exp(-25 * (x - c2[d]) ** 2) for d, x in enumerate(xs)]
    sn = [np.sin(2 * np.pi * x) for x in xs]
    out = np.empty(int(np.prod(shape)), dtype=dtype)
    if len(shape) == 2:
        v = (np.outer(e1[1], e1[0]) + 0.6 * np.outer(e2[1], e2[0])
             + 0.2 * np.outer(sn[1], sn[0]))
        out[:] = v.reshape(-1).astype(dtype)
        return out
    nx, ny, nz = shape
    plane = nx * ny
    a1 = np.outer(e1[1], e1[0])
    a2 = np.outer(e2[1], e2[0])
    a3 = np.outer(sn[1], sn[0])
    for z in range(nz):
        p = e1[2][z] * a1 + 0.6 * e2[2][z] * a2 + 0.2 * sn[2][z] * a3
        out[z * plane:(z + 1) * plane] = p.reshape(-1).astype(dtype)
    return out


def _uniform(n):
    return np.arange(n, dtype=np.float64) / (n - 1)


def _nonuniform(shape):
    out = []
    for d, n in enumerate(shape):
        c = np.cumsum(np.random.default_rng(2105 + d).uniform(0.1, 1.0, n))
        out.append(c / c[-1])
    return out


def _check_classes(plan, got, ref, exact, tol_abs, what):
    """got / ref: device tensors of the flat class buffer."""
    import torch

    for l, s in enumerate(plan.class_slices()):
        if s.stop == s.start:
            continue
        g, r = got[s], ref[s]
        if exact:
            assert torch.equal(g, r), (
                f"{what}: class {l} not bit-identical "
                f"(max |d| = {(g.double() - r.double()).abs().max().item():.3e}, "
                f"{int((g != r).sum().item())} of {g.numel()} differ)")
        else:
            err = (g.double() - r.double()).abs().max().item()
            assert err <= tol_abs, f"{what}: class {l} max|d| {err:.3e} > {tol_abs:.3e}"


def _check_field(got, ref, exact, tol_abs, what):
    import torch

    if exact:
        assert torch.equal(got, ref), (
            f"{what}: not bit-identical (max |d| = "
            f"{(got.double() - ref.double()).abs().max().item():.3e})")
    else:
        err = (got.double() - ref.double()).abs().max().item()
        assert err <= tol_abs, f"{what}: max|d| {err:.3e} > {tol_abs:.3e}"


def _run_config(oracle_mod, shape, dtype, coords, explicit_coords, ks=None,
                expect_levels=None):
    """Both arithmetic policies against ONE oracle run of decompose and of
    recompose at each k."""
    import torch

    from paper_2105_12764_b200 import Plan

    v = _smooth_field_separable(shape, coords, dtype)
    rng_v = float(v.max()) - float(v.min())
    tol_abs = TOL[dtype] * rng_v
    oc = coords if explicit_coords else None
    ref_c, L = oracle_mod.decompose(v, shape, oc)
    if expect_levels is not None:
        assert L == expect_levels
    d_v = torch.from_numpy(v).cuda()
    d_ref = torch.from_numpy(ref_c).cuda()
    ks = sorted(set(ks if ks is not None else (0, L // 2, L)))
    for fast in (False, True):
        plan = Plan(shape, dtype, coords=oc, fast=fast)
        assert plan.levels == L
        got = plan.decompose(d_v)
        _check_classes(plan, got, d_ref, not fast, tol_abs,
                       f"{shape} {dtype} {'fast' if fast else 'exact'} decompose")
        del got
        plan.close()
    for k in ks:
        ref_r = torch.from_numpy(oracle_mod.recompose(ref_c, shape, L, k, oc)).cuda()
        for fast in (False, True):
            plan = Plan(shape, dtype, coords=oc, fast=fast)
            got = plan.recompose(d_ref, k)
            _check_field(got, ref_r, not fast, tol_abs,
                         f"{shape} {dtype} {'fast' if fast else 'exact'} recompose k={k}")
            del got
            plan.close()
        del ref_r
    # lossless round trip of the GPU's own classes (FAST, the benchmarked path)
    plan = Plan(shape, dtype, coords=oc, fast=True)
    back = plan.recompose(plan.decompose(d_v))
    assert (back.double() - d_v.double()).abs().max().item() <= tol_abs
    plan.close()
    del d_v, d_ref, back
    torch.cuda.empty_cache()


def test_config1_65cubed_f64_full(oracle_mod):
    """BASELINE config 1: 65^3 f64 uniform (L = 6); every k."""
    shape = (65, 65, 65)
    coords = [_uniform(n) for n in shape]
    _run_config(oracle_mod, shape, "float64", coords, False, ks=range(7), expect_levels=6)


def test_config2_8193sq_f64_full(oracle_mod):
    """BASELINE config 2: 8193^2 f64 uniform (L = 13): long-fiber Thomas
    (4097 coarse nodes) along both dims."""
    shape = (8193, 8193)
    coords = [_uniform(n) for n in shape]
    _run_config(oracle_mod, shape, "float64", coords, False, expect_levels=13)


def test_config3_513cubed_f32_nonuniform_full(oracle_mod):
    """BASELINE config 3: 513^3 f32, non-uniform coordinates (seeds
    2105..2107, normalized), L = 9."""
    shape = (513, 513, 513)
    coords = _nonuniform(shape)
    _run_config(oracle_mod, shape, "float32", coords, True, expect_levels=9)


def test_config4_1025cubed_f32_full(oracle_mod):
    """BASELINE config 4 (the headline, 1025^3 f32 per GPU, L = 10): rank 0's
    block of the weak-scaling field."""
    shape = (1025, 1025, 1025)
    coords = [(_uniform(n) + 0.0) / 2.0 for n in shape]  # rank 0's block
    _run_config(oracle_mod, shape, "float32", coords, False, expect_levels=10)


def test_config5_block_1025sq_513_f64_full(oracle_mod):
    """BASELINE config 5 block (1025 x 1025 x 513 f64, the global 2049^2 x 1025
    field's block (1, 0, 1), coordinates = the global slices, L = 9)."""
    shape = (1025, 1025, 513)
    g = [_uniform(2049), _uniform(2049), _uniform(1025)]
    coords = [g[0][1024:2049], g[1][0:1025], g[2][512:1025]]
    _run_config(oracle_mod, shape, "float64", coords, True, expect_levels=9)


# ---- cheap shapes that reach the headline configs' kernel instantiations ----
# (17, 9, 1025): 513-long z fibers -> the z solve fused with apply / unapply
#   (thomas_fiber_kernel<R, 2, 33, 32>), as at 1025^3 level 10;
# (8193, 9) / (9, 8193): 4097-long x / y fibers (thomas_cluster_kernel<R,
#   {0,1}, 33, 8>: 8-CTA clusters), as at 8193^2 level 13;
# (4097, 65) / (65, 4097): 2049-long fibers, 4-CTA clusters, 33 fibers (a
#   full and a 1-fiber cluster group);
# (1073, 9) / (9, 1073) / (9, 5, 1073): 537-long fibers, 2-CTA clusters
#   with 17-position chunks (x / y / z);
# (5, 3, 4097): 2049-long z fibers (cluster, DIM 2);
# (1025, 9, 17) / (9, 1025, 17): 513-long x / y fibers.
# FAST y / z fibers of >= 4097 positions go through the two-pass solve
# (thomas_2pass.cuh) instead of the clusters.
TARGETED = [((17, 9, 1025), "float32"), ((17, 9, 1025), "float64"),
            ((8193, 9), "float64"), ((9, 8193), "float64"),
            ((8193, 9), "float32"), ((9, 8193), "float32"),
            ((4097, 65), "float64"), ((65, 4097), "float32"),
            ((1073, 9), "float32"), ((9, 1073), "float64"), ((9, 5, 1073), "float64"),
            ((5, 3, 4097), "float32"),
            ((1025, 9, 17), "float32"), ((9, 1025, 17), "float32"),
            ((33, 17, 2049), "float32"), ((2049, 17, 9), "float64"),
            ((9, 2049, 17), "float64"),
            # non-dyadic long fibers (1501 / 1251 / 1101 coarse positions:
            # partial last chunk of the two-pass solve, thomas_2pass.cuh)
            ((3000, 7), "float64"), ((7, 2500), "float32"), ((5, 3, 2200), "float64"),
            # >= 4097-long y / z fibers: the two-pass solve, incl. a partial
            # last chunk (4501 positions)
            ((7, 9000), "float32"), ((3, 3, 8193), "float64")]


@pytest.mark.parametrize("shape,dtype", TARGETED,
                         ids=lambda x: "x".join(map(str, x)) if isinstance(x, tuple) else x)
@pytest.mark.parametrize("nonuni", [False, True], ids=["uniform", "nonuniform"])
def test_targeted_instantiations(shape, dtype, nonuni, oracle_mod):
    import torch

    from paper_2105_12764_b200 import Plan

    rng = np.random.default_rng(zlib.crc32(repr((shape, dtype, nonuni)).encode()))
    coords = ([np.cumsum(rng.uniform(0.1, 1.0, n)) for n in shape] if nonuni else None)
    v = rng.random(int(np.prod(shape))).astype(dtype)
    tol_abs = TOL[dtype] * float(v.max() - v.min())
    ref_c, L = oracle_mod.decompose(v, shape, coords)
    d_v = torch.from_numpy(v).cuda()
    d_ref = torch.from_numpy(ref_c).cuda()
    for fast in (False, True):
        plan = Plan(shape, dtype, coords=coords, fast=fast)
        assert plan.levels == L
        _check_classes(plan, plan.decompose(d_v), d_ref, not fast, tol_abs,
                       f"{'fast' if fast else 'exact'} decompose")
        for k in sorted({0, L // 2, L - 1, L}):
            ref_r = torch.from_numpy(oracle_mod.recompose(ref_c, shape, L, k, coords)).cuda()
            _check_field(plan.recompose(d_ref, k), ref_r, not fast, tol_abs,
                         f"{'fast' if fast else 'exact'} recompose k={k}")
        plan.close()


@pytest.mark.parametrize("fast", [False, True])
def test_config5_split_decompose_recompose_assemble_downscaled(oracle_mod, fast):
    """Config 5's pipeline on a downscaled field (129x129x65 f64, split 2x2x2
    into 65x65x33 blocks with their global coordinate slices, as bench.py
    --config 5 does at 2049x2049x1025): every block's classes against the
    oracle's decompose of that block (exact policy bit-identical, FAST within
    1e-12 of the range), its full recompose, and the assembled field equal to
    the input (shared planes from the lower block)."""
    import torch

    from paper_2105_12764_b200 import Plan
    from paper_2105_12764_b200 import parallel as par

    shape = (129, 129, 65)
    coords = [_uniform(n) for n in shape]
    v = _smooth_field_separable(shape, coords, np.float64)
    rng = float(v.max() - v.min())
    specs = par.split_blocks(shape, (2, 2, 2))
    assert [s.shape for s in specs] == [(65, 65, 33)] * 8
    rec_blocks = {}
    for sp in specs:
        g = par.block_grid(v, shape, coords, sp)
        plan = Plan(sp.shape, "float64", coords=g.coords, device=0, fast=fast)
        d = torch.from_numpy(g.values).cuda()
        c = plan.decompose(d)
        ref_c, L = oracle_mod.decompose(g.values, sp.shape, g.coords)
        assert L == plan.levels
        got = c.cpu().numpy()
        if fast:
            assert float(np.abs(got - ref_c).max()) <= 1e-12 * rng
        else:
            assert np.array_equal(got, ref_c)
        rec_blocks[sp.index] = plan.recompose(c).cpu().numpy()
        plan.close()
    back = par.assemble_blocks(rec_blocks, specs, shape)
    assert float(np.abs(back - v).max()) <= 1e-12 * rng
