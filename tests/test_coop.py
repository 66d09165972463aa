"""Cooperative multi-GPU decompose (SURVEY.md §8(f) row 3,
parallel_impl.hpp:691-808): partition rules (CPU, mirroring
test_parallel.cpp:32-86), slab/class-fragment bookkeeping (CPU), the
send/recv transport on a 2-process gloo group (CPU), and the device path
with W workers on one GPU, bit-identical to the serial decompose
(test_parallel.cpp:88-123)."""
import os
import socket
import sys
import zlib

import numpy as np
import pytest

from paper_2105_12764_b200 import coop, errors

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


# ---- partitions (parallel.cpp:9-90) -----------------------------------------
def test_one_worker_owns_the_grid():
    p = coop.make_partitions((9, 9, 9), 1, coop.PartitionScheme.block)
    assert len(p) == 1 and p[0].lo == (0, 0, 0) and p[0].hi == (9, 9, 9)


def test_block_slabs_slowest_dimension():
    p = coop.make_partitions((9, 9, 9), 3, coop.PartitionScheme.block)
    assert [(q.worker, q.lo[2], q.hi[2]) for q in p] == [(0, 0, 3), (1, 3, 6), (2, 6, 9)]
    assert all(q.lo[0] == 0 and q.hi[0] == 9 for q in p)


def test_shifted_round_robin_is_cyclic():
    p = coop.make_partitions((9, 9), 3, coop.PartitionScheme.shifted_round_robin)
    assert len(p) == 9
    for s in range(2):
        for stage in range(3):
            assert len({q.worker for q in p if q.block_coord[s] == stage}) == 3
    assert all(q.worker == (q.block_coord[0] + q.block_coord[1]) % 3 for q in p)


def test_partition_validation():
    with pytest.raises(errors.TooManyWorkers):
        coop.make_partitions((9, 9), 10, coop.PartitionScheme.block)
    with pytest.raises(errors.TooManyWorkers):
        coop.make_partitions((9, 9), 10, coop.PartitionScheme.shifted_round_robin)
    with pytest.raises(errors.ShapeError):
        coop.make_partitions((9,), 2, coop.PartitionScheme.shifted_round_robin)
    with pytest.raises(errors.TooManyWorkers):
        coop.make_partitions((9,), 0, coop.PartitionScheme.block)


# ---- slab bookkeeping -------------------------------------------------------
def _level_shapes(shape):
    import oracle

    L, ext = oracle.hierarchy(shape)
    return [tuple(int(x) for x in e) for e in ext]


@pytest.mark.parametrize("shape,workers", [((33, 33, 33), 2), ((33, 33, 33), 4),
                                           ((17, 17, 17), 3), ((65, 33, 129), 5),
                                           ((1025, 1025, 1025), 8), ((9, 9, 9), 2)])
def test_slabs_and_fragments_partition_every_level(shape, workers):
    ls = _level_shapes(shape)
    L = len(ls) - 1
    q = coop.coop_levels(ls, workers)
    assert q >= 1
    b = coop.slab_bounds(shape[2], workers, q)
    assert b[0] == 0 and b[-1] == shape[2] - 1 and all(x % (1 << q) == 0 for x in b[:-1])
    for j in range(q):
        l = L - j
        m2 = ls[l - 1][2]
        rng = [coop.coarse_range(b, r, j, m2) for r in range(workers)]
        assert rng[0][0] == 0 and rng[-1][1] == m2
        assert all(rng[r][1] == rng[r + 1][0] and rng[r][0] < rng[r][1]
                   for r in range(workers - 1))
        # class-l fragments tile class l exactly once
        F, C = int(np.prod(ls[l])), int(np.prod(ls[l - 1]))
        cover = np.zeros(F - C, dtype=np.int32)
        for c0, c1 in rng:
            for o, n in coop.class_pieces(ls[l], c0, c1, m2):
                cover[o:o + n] += 1
        assert (cover == 1).all()


def test_non_cooperative_shapes():
    assert coop.coop_levels(_level_shapes((12, 10, 9)), 2) == 0  # even extents
    assert coop.coop_levels(_level_shapes((33, 33)), 2) == 0     # 2-D
    assert coop.coop_levels(_level_shapes((33, 33, 5)), 8) == 0  # too few planes


# ---- transport on a real 2-process group (gloo, CPU tensors) ---------------
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _transport_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tp = coop.DistTransport()
        buf = torch.full((8,), float(rank))
        pairs = [(0, buf[0:2] if rank == 0 else None, 1, buf[4:6] if rank == 1 else None),
                 (1, buf[2:4] if rank == 1 else None, 0, buf[6:8] if rank == 0 else None)]
        rep = coop.CommReport()
        tp.move(pairs, rep, "halo")
        q.put((rank, buf.tolist(), rep.phases["halo"].elements))
    finally:
        dist.destroy_process_group()


def test_dist_transport_gloo_two_ranks():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_transport_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict((r, (b, n)) for r, b, n in (q.get(timeout=120) for _ in ps))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[1][0] == [1, 1, 1, 1, 0, 0, 1, 1]
    assert out[0][0] == [0, 0, 0, 0, 0, 0, 1, 1]
    assert out[0][1] == 4 and out[1][1] == 4


# ---- device path: W workers on one GPU, bit-identical to serial --------------
@pytest.mark.gpu
@pytest.mark.parametrize("shape,workers", [((17, 17, 17), 2), ((17, 17, 17), 3),
                                           ((17, 17, 17), 4), ((33, 33, 33), 2),
                                           ((33, 17, 65), 5), ((65, 65, 65), 8),
                                           ((9, 9, 9), 1), ((12, 10, 9), 3)])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("nonuni", [False, True], ids=["uniform", "nonuniform"])
def test_cooperative_equals_serial(shape, workers, dtype, nonuni):
    from paper_2105_12764_b200 import decompose, make_grid

    rng = np.random.default_rng(zlib.crc32(repr((shape, workers, dtype, nonuni)).encode()))
    coords = [np.cumsum(rng.uniform(0.1, 1.0, n)) for n in shape] if nonuni else None
    g = make_grid(shape, rng.random(int(np.prod(shape))).astype(dtype), coords)
    serial = decompose(g)
    rep = coop.CommReport()
    r = coop.cooperative_decompose(g, workers, coop.CoopOptions(report=rep),
                                   transport=coop.LocalTransport(workers))
    assert r.levels == serial.levels
    for l in range(r.levels + 1):
        assert np.array_equal(np.asarray(r.classes[l]), np.asarray(serial.classes[l])), l
    split = workers > 1 and coop.coop_levels(
        [tuple(int(x) for x in e) for e in _level_shapes(shape)], workers)
    if split:
        assert rep.phases["classes"].elements > 0
    # the native runtime (csrc/coop_host.cuh): same classes
    nrep = coop.CommReport()
    n = coop.cooperative_decompose(g, workers, coop.CoopOptions(report=nrep))
    assert np.array_equal(np.asarray(n.flat), np.asarray(serial.flat))
    assert (nrep.phases["native"].elements > 0) == bool(split)


@pytest.mark.gpu
def test_cooperative_level_cap_and_fast_policy():
    from paper_2105_12764_b200 import RefactorOptions, decompose, make_grid

    rng = np.random.default_rng(5)
    g = make_grid((33, 33, 65), rng.random(33 * 33 * 65).astype("float32"))
    serial = decompose(g, RefactorOptions(levels=3))
    r = coop.cooperative_decompose(g, 4, coop.CoopOptions(levels=3),
                                   transport=coop.LocalTransport(4))
    nat = coop.cooperative_decompose(g, 4, coop.CoopOptions(levels=3))
    assert np.array_equal(np.asarray(nat.flat), np.asarray(serial.flat))
    assert r.levels == 3
    assert all(np.array_equal(np.asarray(a), np.asarray(b))
               for a, b in zip(r.classes, serial.classes))
    f = coop.cooperative_decompose(g, 4, coop.CoopOptions(fast=True))
    ref = decompose(g)
    rg = float(g.values.max() - g.values.min())
    for a, b in zip(f.classes, ref.classes):
        assert np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)).max() <= 1e-5 * rg


@pytest.mark.gpu
def test_cooperative_fault_injection_is_worker_failure():
    from paper_2105_12764_b200 import make_grid

    g = make_grid((17, 17, 17), np.zeros(17 ** 3))

    def boom(w, phase, level):
        if w == 1 and phase == "solve":
            raise RuntimeError("injected")

    with pytest.raises(errors.WorkerFailure):
        coop.cooperative_decompose(g, 2, coop.CoopOptions(fault_injector=boom),
                                   transport=coop.LocalTransport(2))
    with pytest.raises(errors.WorkerFailure):  # native runtime, C callback
        coop.cooperative_decompose(g, 2, coop.CoopOptions(fault_injector=boom))


def _coop_rank(rank, world, port, q, shape, dtype):
    import torch
    import torch.distributed as dist

    from paper_2105_12764_b200 import make_grid

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        rng = np.random.default_rng(11)
        g = make_grid(shape, rng.random(int(np.prod(shape))).astype(dtype))
        r = coop.cooperative_decompose(g, world, coop.CoopOptions(batches=3),
                                       transport=coop.DistTransport())
        q.put((rank, None if r is None else r.flat))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_cooperative_over_process_group(world):
    """One worker per torch.distributed rank (the multi-GPU code path: halo,
    pipelined z-solve over 3 fiber batches, gathers), here W processes on one
    GPU over gloo; rank 0's classes equal the serial decompose bit for bit."""
    import torch.multiprocessing as mp

    from paper_2105_12764_b200 import decompose, make_grid

    shape, dtype = (33, 17, 65), "float64"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_coop_rank, args=(r, world, port, q, shape, dtype))
          for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(11)
    g = make_grid(shape, rng.random(int(np.prod(shape))).astype(dtype))
    serial = decompose(g)
    assert np.array_equal(out[0], np.asarray(serial.flat))
    assert all(out[r] is None for r in range(1, world))


@pytest.mark.gpu
def test_grouped_decompose_equals_serial_per_block():
    """test_parallel.cpp:225-240."""
    from paper_2105_12764_b200 import decompose, grouped_decompose, make_grid

    rng = np.random.default_rng(80)
    blocks = [make_grid((17, 17, 17), rng.random(17 ** 3)) for _ in range(4)]
    res = grouped_decompose(blocks, 2, 2)
    assert len(res) == 4
    for b, r in zip(blocks, res):
        assert np.array_equal(np.asarray(r.flat), np.asarray(decompose(b).flat))
    one = [make_grid((9, 9), rng.random(81))]
    g = grouped_decompose(one, 1, 1)
    c = coop.cooperative_decompose(one[0], 1)
    assert np.array_equal(np.asarray(g[0].flat), np.asarray(c.flat))
    with pytest.raises(errors.TooManyWorkers):
        grouped_decompose(one, 0, 1)
