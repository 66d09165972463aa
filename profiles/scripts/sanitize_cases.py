"""Small decompose / recompose / unit-kernel / container / compress / coop
cases covering every kernel family, for compute-sanitizer runs
(profiles/scripts/sanitize.sh).  Each case also checks its values against the
oracle so a sanitizer-perturbed run that computes garbage is visible.

  compute-sanitizer --tool memcheck python profiles/scripts/sanitize_cases.py
"""
import os
import sys
import tempfile

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (checker)
from paper_2105_12764_b200 import Plan  # noqa: E402

rng = np.random.default_rng(7)
dev = torch.device("cuda", 0)
quick = os.environ.get("SAN_QUICK") == "1"

# (shape, dtype, nonuniform, fast): lean dyadic (both policies, f32/f64),
# non-dyadic pair-lane / generic 3-D, 2-D, 1-D, extent-2 dims, long fibers
# (chunked Thomas variants), 4-D generic path.
CASES = [
    ((33, 17, 9), "float32", False, True),
    ((33, 17, 9), "float32", False, False),
    ((17, 9, 33), "float64", True, True),
    ((17, 9, 33), "float64", True, False),
    ((65, 33, 17), "float32", False, True),
    ((20, 13, 10), "float32", False, False),
    ((20, 13, 10), "float64", True, True),
    ((12, 7, 6), "float64", False, False),
    ((257, 129), "float64", False, True),
    ((257, 129), "float64", False, False),
    ((100, 37), "float32", True, False),
    ((1025,), "float64", False, True),
    ((1000,), "float32", False, False),
    ((2, 9, 5), "float32", False, False),
    ((17, 9, 1025), "float32", False, True),
    ((2049, 9), "float64", False, True),
    ((9, 2049), "float64", False, True),
    ((9, 7, 5, 5), "float32", False, False),
    ((9, 9, 5, 3), "float64", True, True),
    # round 2: long fibers on thread-block clusters (DSMEM carries), 8-warp
    # f64 y / z CTAs
    ((8193, 9), "float64", False, True),
    ((9, 4097), "float32", True, True),
    ((9, 1073), "float64", False, True),
    ((9, 5, 1073), "float64", True, True),
    ((5, 3, 4097), "float32", False, True),
    ((33, 65, 257), "float64", False, True),
    # round 2 (late): two-pass long strided fibers (thomas_2pass.cuh), DIM 1
    # and DIM 2, incl. a partial last chunk
    ((9, 8193), "float64", False, True),
    ((3, 3, 8193), "float32", True, True),
    ((7, 9000), "float32", False, True),
]
NEW = CASES[-3:]
if quick:
    CASES = CASES[:4] + CASES[8:9] + CASES[17:18]


def run_case(shape, dt, nonuni, fast):
    coords = ([np.cumsum(rng.uniform(0.1, 1.0, n)) for n in shape] if nonuni else None)
    v = rng.random(int(np.prod(shape))).astype(dt)
    plan = Plan(shape, dt, coords=coords, device=0, fast=fast)
    d_v = torch.from_numpy(v).to(dev)
    d_c = plan.decompose(d_v)
    L = plan.levels
    outs = [plan.recompose(d_c, k) for k in sorted({0, L // 2, L})]
    torch.cuda.synchronize()
    ref_c, Lr = oracle.decompose(v, shape, coords)
    assert Lr == L
    got = d_c.cpu().numpy()
    if fast:
        tol = (1e-5 if dt == "float32" else 1e-12) * float(v.max() - v.min())
        assert float(np.abs(got.astype(np.float64) - ref_c).max()) <= tol, shape
    else:
        assert np.array_equal(got, ref_c), shape
        for k, o in zip(sorted({0, L // 2, L}), outs):
            assert np.array_equal(o.cpu().numpy(), oracle.recompose(ref_c, shape, L, k, coords))
    # unit-kernel entry points on the finest level (GPK / mass-trans / solve)
    if len(shape) <= 3 and L >= 1:
        lv = L
        n = int(np.prod(plan.level_shape(lv)))
        x = torch.from_numpy(rng.random(n).astype(dt)).to(dev)
        plan.gpk(lv, x.clone())
        plan.gpk(lv, x.clone(), inverse=True)
        torch.cuda.synchronize()
    # container write/read + CRC, and one compress/decompress round
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "f.mgrf")
        plan.write_refactored(d_c, p)
        plan.read_refactored(p)
    blob = plan.compress(d_v, 1e-3)
    plan.decompress(blob[0] if isinstance(blob, tuple) else blob)
    torch.cuda.synchronize()
    plan.close()


def run_coop():
    from paper_2105_12764_b200 import coop, refactor

    shape = (33, 33, 33)
    v = rng.random(int(np.prod(shape))).astype(np.float32)
    g = refactor.make_grid(shape, v)
    r = coop.cooperative_decompose(g, 2)
    ref_c, _ = oracle.decompose(v, shape)
    flat = np.concatenate([np.asarray(c).reshape(-1) for c in r.classes])
    assert np.array_equal(flat, ref_c)


def run_host(shape, dt, fast):
    """Host-buffer entry points: pageable (pinned rings + download worker,
    csrc/hostio.cuh) and per-class buffers; the pipelined path at >= 2^22
    nodes."""
    import ctypes

    from paper_2105_12764_b200 import _lib

    v = rng.random(int(np.prod(shape))).astype(dt)
    plan = Plan(shape, dt, device=0, fast=fast)
    ref = plan.decompose(torch.from_numpy(v).to(dev)).cpu().numpy()
    sl = plan.class_slices()
    cls = [np.empty(s.stop - s.start, dtype=dt) for s in sl]
    ptrs = (ctypes.c_void_p * len(cls))(*[c.ctypes.data for c in cls])
    _lib.check(_lib.lib().mgrg_decompose_host_classes(plan._h, v.ctypes.data, ptrs))
    assert np.array_equal(np.concatenate(cls), ref)
    back = np.empty_like(v)
    _lib.check(_lib.lib().mgrg_recompose_host_classes(plan._h, ptrs, plan.levels,
                                                      back.ctypes.data))
    flat = np.empty_like(v)
    _lib.check(_lib.lib().mgrg_decompose_host(plan._h, v.ctypes.data, flat.ctypes.data))
    assert np.array_equal(flat, ref)
    plan.close()


def run_crc():
    """GPU CRC-32 on a range long enough for the lane-private-table kernel
    (>= 2^16 blocks) plus the tree combine, against zlib."""
    import zlib

    from paper_2105_12764_b200 import crc32

    n = (1 << 16) * 512 + 4 * 1000 + 12  # + a partial segment and a tail
    x = torch.from_numpy(rng.integers(0, 256, n, dtype=np.uint8)).to(dev)
    for a in (0, 5):
        assert crc32(x[a:]) == zlib.crc32(x[a:].cpu().numpy().tobytes())


only_new = os.environ.get("SAN_ONLY_NEW") == "1"
for c in (NEW if only_new else CASES):
    run_case(*c)
    print("ok", c, flush=True)
run_crc()
print("ok crc", flush=True)
if only_new:
    sys.exit(0)
for shp, dt, fast in (((129, 129, 257), "float32", True), ((129, 129, 257), "float32", False),
                      ((33, 17, 9), "float64", True)):
    run_host(shp, dt, fast)
    print("ok host", shp, dt, fast, flush=True)
run_coop()
print("ok coop", flush=True)
print("sanitize cases done", flush=True)
