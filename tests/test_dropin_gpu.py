"""Drop-in contract details of the Python API and the C ABI that need a
GPU: PassStats through decompose AND recompose against the reference
engine's counters (acceptance criterion 9, acceptance.cpp:336-374); class
arrays replaced after decompose are what recompose / write_refactored use
(the reference treats classes as the data); tensors on the wrong device are
rejected; the block metadata record (GPU CRC) and the native NCCL all-gather
(world size 1 on one GPU -- the multi-rank path is the same call)."""
import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _stats_as_dicts(st):
    def pc(c):
        return (c.in_, c.out)

    return [{"level": lv.level, "level_elements": lv.level_elements,
             "coefficient": pc(lv.coefficient), "fused_copy": pc(lv.fused_copy),
             "masstrans": [pc(c) for c in lv.masstrans], "solve": [pc(c) for c in lv.solve],
             "apply": pc(lv.apply)} for lv in st.levels]


@pytest.mark.parametrize("shape,nonuni,cap", [((17, 17, 17), False, 0), ((12, 10, 9), False, 0),
                                              ((33, 17), True, 0), ((65,), False, 3),
                                              ((9, 5, 3, 6), True, 0)])
def test_pass_stats_decompose_and_recompose_match_reference(oracle_mod, shape, nonuni, cap):
    if not oracle_mod.available("ref"):
        pytest.skip("oracle/_ref not built")
    from paper_2105_12764_b200 import refactor as R

    rng = np.random.default_rng(9000)
    coords = ([np.cumsum(rng.uniform(0.1, 1.0, n)) for n in shape] if nonuni else None)
    v = rng.random(int(np.prod(shape)))
    g = R.make_grid(shape, v, coords)
    st = R.PassStats()
    opt = R.RefactorOptions(levels=cap or None, stats=st)
    r = R.decompose(g, opt)
    assert _stats_as_dicts(st) == oracle_mod.ref_pass_stats(v, shape, coords, cap)
    R.recompose(r, r.levels, opt)
    assert _stats_as_dicts(st) == oracle_mod.ref_pass_stats(v, shape, coords, cap,
                                                            recompose=True)


@pytest.mark.parametrize("host", [True, False])
def test_replaced_class_arrays_are_used(oracle_mod, host):
    import torch

    from paper_2105_12764_b200 import container, refactor as R

    shape = (17, 9, 9)
    v = np.random.default_rng(1).random(int(np.prod(shape)))
    vals = v if host else torch.from_numpy(v).cuda()
    r = R.decompose(R.make_grid(shape, vals))
    L = r.levels
    # zero the finest class in place of the original array (a quantizer would)
    r.classes[L] = np.zeros_like(r.classes[L]) if host else torch.zeros_like(r.classes[L])
    got = R.recompose(r, L).values
    got = got if host else got.cpu().numpy()
    ref_c, _ = oracle_mod.decompose(v, shape)
    offs = oracle_mod.class_offsets(shape, L)
    ref_c[offs[L]:offs[L + 1]] = 0
    assert np.array_equal(got, oracle_mod.recompose(ref_c, shape, L, L))
    # and a container written from it holds the replaced class
    import tempfile, os
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "z.mgrf")
        container.write_refactored(r, p)
        back = container.read_refactored(p)
        cl = back.data.classes[L]
        cl = cl.cpu().numpy() if hasattr(cl, "cpu") else np.asarray(cl)
        assert not cl.any()


def test_wrong_device_and_noncontiguous_tensors_rejected():
    import torch

    from paper_2105_12764_b200 import Plan, errors

    plan = Plan((17, 9), "float64", device=0)
    with pytest.raises(errors.InvalidArgument):
        plan.decompose(torch.zeros(17 * 9, dtype=torch.float64))  # host tensor
    x = torch.zeros(9, 17 * 2, dtype=torch.float64, device="cuda")[:, ::2]
    with pytest.raises(errors.InvalidArgument):
        plan.decompose(x.reshape(-1) if x.is_contiguous() else x.t())
    plan.close()


def test_block_meta_and_native_allgather_world1():
    import torch

    from paper_2105_12764_b200 import Plan, parallel

    shape = (33, 17, 9)
    v = torch.rand(int(np.prod(shape)), dtype=torch.float32, device="cuda")
    plan = Plan(shape, "float32", device=0)
    c = plan.decompose(v)
    m = parallel.block_meta(plan, c, block=3, rank=0, origin=(32, 0, 8),
                            decompose_ms=1.5, recompose_ms=2.25)
    host = c.cpu().numpy()
    offs = plan.class_offsets
    crcs = [zlib.crc32(host[offs[l]:offs[l + 1]].view(np.uint8)) for l in range(plan.levels + 1)]
    assert m.class_crc32 == crcs
    assert m.class_bytes == [4 * (offs[l + 1] - offs[l]) for l in range(plan.levels + 1)]
    le = b"".join(int(x).to_bytes(4, "little") for x in crcs)
    assert m.checksum == zlib.crc32(le)
    assert m.origin == (32, 0, 8) and m.shape == shape and m.levels == plan.levels
    comm = parallel.NativeMetaComm(0, 1, 0, parallel.NativeMetaComm.unique_id())
    other = parallel.BlockMeta(block=1, rank=0, origin=(0, 0, 0), shape=shape, dtype_bytes=4,
                               levels=m.levels, class_bytes=m.class_bytes,
                               class_crc32=m.class_crc32, decompose_us=10, recompose_us=20)
    got = comm.allgather([m, other], per_rank=3)  # one padding record
    assert [g.block for g in got] == [1, 3]
    assert got[1].class_crc32 == m.class_crc32 and got[1].decompose_us == 1500
    assert got[0].recompose_us == 20
    comm.close()
    plan.close()


def test_coop_schedule_matches_runtime_rule():
    import ctypes

    from paper_2105_12764_b200 import Plan, _lib, coop

    plan = Plan((33, 33, 33), "float64", device=0)
    q = ctypes.c_int32(0)
    bounds = (ctypes.c_uint64 * 3)()
    _lib.check(_lib.lib().mgrg_coop_schedule(plan._h, 2, ctypes.byref(q), bounds))
    shapes = [plan.level_shape(l) for l in range(plan.levels + 1)]
    assert q.value == coop.coop_levels(shapes, 2) == 4
    assert list(bounds) == coop.slab_bounds(33, 2, 4) == [0, 16, 32]
    n = ctypes.c_int32(0)
    _lib.check(_lib.lib().mgrg_device_count(ctypes.byref(n)))
    assert n.value >= 1
    plan.close()


@pytest.mark.parametrize("shape,dt,fast", [((65, 33, 17), "float32", True),
                                           ((33, 17, 9), "float64", False),
                                           ((257, 129), "float64", True),
                                           ((9, 8193), "float64", True)])  # two-pass solve
def test_graph_replay_identical(shape, dt, fast):
    """mgrg_plan_set_graphs: captured-graph replay gives the same bits as the
    stream launches, for repeated calls, a second buffer set (new capture)
    and every classes_used."""
    import torch

    from paper_2105_12764_b200 import Plan

    v = torch.rand(int(np.prod(shape)), dtype=getattr(torch, dt), device="cuda")
    plan = Plan(shape, dt, fast=fast)
    c0 = plan.decompose(v)
    r0 = [plan.recompose(c0, k) for k in range(plan.levels + 1)]
    plan.set_graphs(True)
    c1 = torch.empty_like(c0)
    for _ in range(3):
        plan.decompose(v, c1)
        assert torch.equal(c1, c0)
    v2 = v.clone()
    c2 = plan.decompose(v2)
    assert torch.equal(c2, c0)
    out = torch.empty_like(v)
    for k in range(plan.levels + 1):
        for _ in range(2):
            plan.recompose(c1, k, out)
            assert torch.equal(out, r0[k])
    assert plan.last_launches > 0
    plan.set_graphs(False)
    plan.close()


# ---- host-buffer entry points: pageable vs pinned, flat vs per-class ---------
# (csrc/hostio.cuh).  (129, 129, 257) has 4.3M nodes: the pipelined host paths
# (dyadic 3-D, >= 2^22 nodes) in both policies; (33, 17, 9) the plain path.
@pytest.mark.parametrize("shape", [(129, 129, 257), (33, 17, 9)], ids=["pipelined", "plain"])
@pytest.mark.parametrize("fast", [False, True], ids=["exact", "fast"])
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_host_entry_points_pageable_pinned_per_class(shape, fast, dtype):
    import ctypes

    import torch

    from paper_2105_12764_b200 import Plan, _lib

    rng = np.random.default_rng(zlib.crc32(repr((shape, fast, dtype)).encode()))
    v = rng.random(int(np.prod(shape))).astype(dtype)
    plan = Plan(shape, dtype, fast=fast, device=0)
    L = plan.levels
    ref = plan.decompose(torch.from_numpy(v).cuda()).cpu().numpy()
    ref_r = {k: plan.recompose(torch.from_numpy(ref).cuda(), k).cpu().numpy()
             for k in (L - 1, L)}
    lib = _lib.lib()
    # pageable flat buffers
    out = np.full_like(v, np.nan)
    _lib.check(lib.mgrg_decompose_host(plan._h, v.ctypes.data, out.ctypes.data))
    assert np.array_equal(out, ref)
    # pinned flat buffers (torch pinned host tensors)
    pin_in = torch.from_numpy(v).pin_memory()
    pin_out = torch.empty_like(pin_in).pin_memory()
    _lib.check(lib.mgrg_decompose_host(plan._h, pin_in.data_ptr(), pin_out.data_ptr()))
    assert np.array_equal(pin_out.numpy(), ref)
    # per-class pageable buffers, written in place
    sl = plan.class_slices()
    cls = [np.full(s.stop - s.start, np.nan, dtype=dtype) for s in sl]
    ptrs = (ctypes.c_void_p * len(cls))(*[c.ctypes.data for c in cls])
    _lib.check(lib.mgrg_decompose_host_classes(plan._h, v.ctypes.data, ptrs))
    for s, c in zip(sl, cls):
        assert np.array_equal(c, ref[s])
    # recompose from per-class pageable buffers (k = L: pipelined; k = L-1: prefix)
    for k in (L - 1, L):
        back = np.full_like(v, np.nan)
        _lib.check(lib.mgrg_recompose_host_classes(plan._h, ptrs, k, back.ctypes.data))
        assert np.array_equal(back, ref_r[k]), f"recompose_host_classes k={k}"
        back2 = np.full_like(v, np.nan)
        _lib.check(lib.mgrg_recompose_host(plan._h, ref.ctypes.data, k, back2.ctypes.data))
        assert np.array_equal(back2, ref_r[k]), f"recompose_host k={k}"
    # classes above k are never read: null pointers there are accepted
    ptrs_k = (ctypes.c_void_p * len(cls))(*([c.ctypes.data for c in cls[:L]] + [None]))
    back = np.full_like(v, np.nan)
    _lib.check(lib.mgrg_recompose_host_classes(plan._h, ptrs_k, L - 1, back.ctypes.data))
    assert np.array_equal(back, ref_r[L - 1])
    plan.close()


def test_host_classes_entry_points_reject_null_class():
    import ctypes

    from paper_2105_12764_b200 import Plan, _lib, errors

    shape = (17, 9, 9)
    plan = Plan(shape, "float64", device=0)
    v = np.random.default_rng(3).random(int(np.prod(shape)))
    sl = plan.class_slices()
    cls = [np.empty(s.stop - s.start) for s in sl]
    ptrs = (ctypes.c_void_p * len(cls))(*([c.ctypes.data for c in cls[:-1]] + [None]))
    with pytest.raises(errors.Error):
        _lib.check(_lib.lib().mgrg_decompose_host_classes(plan._h, v.ctypes.data, ptrs))
    plan.close()


def test_host_entry_points_reject_device_pointers():
    import torch

    from paper_2105_12764_b200 import Plan, _lib, errors

    shape = (17, 9, 9)
    plan = Plan(shape, "float32", device=0)
    d = torch.rand(int(np.prod(shape)), device="cuda")
    h = np.empty(int(np.prod(shape)), dtype=np.float32)
    with pytest.raises(errors.Error, match="device pointer"):
        _lib.check(_lib.lib().mgrg_decompose_host(plan._h, d.data_ptr(), h.ctypes.data))
    with pytest.raises(errors.Error, match="device pointer"):
        _lib.check(_lib.lib().mgrg_recompose_host(plan._h, h.ctypes.data, plan.levels,
                                                  d.data_ptr()))
    plan.close()


@pytest.mark.parametrize("shape", [(129, 129, 257), (33, 17, 9)], ids=["large", "small"])
def test_split_host_calls(shape):
    """mgrg_*_host_begin / _end (the drop-in allocates its outputs in between)
    equal the one-shot host calls; misuse is InvalidArgument; abort clears."""
    import ctypes

    import torch

    from paper_2105_12764_b200 import Plan, _lib, errors

    lib = _lib.lib()
    rng = np.random.default_rng(11)
    v = rng.random(int(np.prod(shape))).astype(np.float32)
    plan = Plan(shape, "float32", fast=True, device=0)
    L = plan.levels
    ref = plan.decompose(torch.from_numpy(v).cuda()).cpu().numpy()
    sl = plan.class_slices()
    cls = [np.full(s.stop - s.start, np.nan, dtype=np.float32) for s in sl]
    ptrs = (ctypes.c_void_p * len(cls))(*[c.ctypes.data for c in cls])
    _lib.check(lib.mgrg_decompose_host_begin(plan._h, v.ctypes.data))
    with pytest.raises(errors.Error, match="already in flight"):
        _lib.check(lib.mgrg_decompose_host_begin(plan._h, v.ctypes.data))
    _lib.check(lib.mgrg_decompose_host_end(plan._h, ptrs))
    assert np.array_equal(np.concatenate(cls), ref)
    with pytest.raises(errors.Error, match="no mgrg_decompose_host_begin"):
        _lib.check(lib.mgrg_decompose_host_end(plan._h, ptrs))
    for k in (L - 1, L):
        want = plan.recompose(torch.from_numpy(ref).cuda(), k).cpu().numpy()
        out = np.full_like(v, np.nan)
        _lib.check(lib.mgrg_recompose_host_begin(plan._h, ptrs, k))
        _lib.check(lib.mgrg_recompose_host_end(plan._h, out.ctypes.data))
        assert np.array_equal(out, want)
    # abandoned split call: abort, then the plan is usable again
    _lib.check(lib.mgrg_recompose_host_begin(plan._h, ptrs, L))
    _lib.check(lib.mgrg_host_abort(plan._h))
    out = np.empty_like(v)
    _lib.check(lib.mgrg_recompose_host(plan._h, ref.ctypes.data, L, out.ctypes.data))
    plan.close()


def test_two_pass_solve_launch_count():
    """A FAST y solve of >= 4097 positions runs as three kernels (pass 1,
    carry scan, pass 2: csrc/thomas_2pass.cuh) and the plan's launch count
    includes them: one profile record per counted launch, plus two for the
    (9, 8193) decompose's single two-pass solve (the top level's y fibers)."""
    import torch

    from paper_2105_12764_b200 import Plan

    v = torch.rand(9 * 8193, dtype=torch.float64, device="cuda")
    plan = Plan((9, 8193), "float64", fast=True)
    c = plan.decompose(v)
    plan.set_profiling(True)
    plan.decompose(v, c)
    torch.cuda.synchronize()
    recs = plan.profile(reset=True)
    # one profile record per counted solve / level kernel; the top level's y
    # solve (m = 4097) adds two kernels to the count
    assert plan.last_launches == len(recs) + 2
    plan.close()
