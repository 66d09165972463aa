"""Host logic of the block-sharded multi-GPU path, on CPU:
block splitting / assembly with shared planes,
round-robin dealing, metadata records, and the one collective -- the
metadata all-gather -- over a world-size-2 gloo group (the NCCL path runs
the same code on CUDA tensors).  Block results are produced by the CPU
oracle (test infrastructure) standing in for the device decompose."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2105_12764_b200 import errors
from paper_2105_12764_b200.parallel import (BlockMeta, BlockShardedRefactor, assemble_blocks,
                                            assign_blocks, class_crc32, extract_block,
                                            split_blocks, split_points)
from paper_2105_12764_b200.refactor import RefactoredData


def test_split_points_config5():
    assert split_points(2049, 2) == [0, 1024, 2048]
    assert split_points(1025, 2) == [0, 512, 1024]
    assert split_points(10, 3) == [0, 3, 6, 9]
    with pytest.raises(errors.InvalidGrid):
        split_points(2, 2)


def test_split_blocks_config5_geometry():
    specs = split_blocks((2049, 2049, 1025), (2, 2, 2))
    assert len(specs) == 8
    for s in specs:
        assert s.shape == (1025, 1025, 513)
        bx, by, bz = s.index & 1, (s.index >> 1) & 1, s.index >> 2
        assert s.origin == (1024 * bx, 1024 * by, 512 * bz)


def test_split_assemble_roundtrip():
    shape = (9, 7, 5)
    v = np.arange(int(np.prod(shape)), dtype=np.float64)
    specs = split_blocks(shape, (2, 3, 2))
    blocks = {s.index: extract_block(v, shape, s) for s in specs}
    assert np.array_equal(assemble_blocks(blocks, specs, shape), v)


def test_assemble_takes_shared_planes_from_lower_block():
    shape = (5, 3)
    specs = split_blocks(shape, (2, 1))
    blocks = {0: np.zeros(9), 1: np.ones(9)}
    out = assemble_blocks(blocks, specs, shape).reshape(3, 5)
    assert np.all(out[:, 2] == 0.0)  # shared column x = 2 from block 0
    assert np.all(out[:, 3:] == 1.0)


def test_assign_blocks_round_robin():
    assert assign_blocks(8, 0, 3) == [0, 3, 6]
    assert assign_blocks(8, 2, 3) == [2, 5]
    assert sorted(sum((assign_blocks(8, r, 4) for r in range(4)), [])) == list(range(8))
    with pytest.raises(errors.TooManyWorkers):
        assign_blocks(8, 4, 4)


def test_meta_pack_roundtrip():
    m = BlockMeta(block=5, rank=1, origin=(1024, 0, 512), shape=(1025, 1025, 513),
                  dtype_bytes=8, levels=9, class_bytes=list(range(10, 20)),
                  class_crc32=list(range(100, 110)), decompose_us=1234, recompose_us=99)
    assert BlockMeta.unpack(m.pack()) == m


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shape = (17, 17, 9)
        specs = split_blocks(shape, (2, 2, 1))
        field = oracle.smooth_field(shape)
        sh = BlockShardedRefactor(len(specs))
        for i in sh.mine:
            s = specs[i]
            v = extract_block(field, shape, s)
            cls, L = oracle.decompose(v, s.shape)
            off = oracle.class_offsets(s.shape, L)
            r = RefactoredData(s.shape, None, L, [cls[off[l]:off[l + 1]] for l in range(L + 1)])
            sh.record(i, s, r, 8)
        metas = sh.finish()
        q.put((rank, sh.mine, [m.pack().tolist() for m in metas]))
    finally:
        dist.destroy_process_group()


def test_metadata_allgather_gloo_world2(oracle_mod):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == [0, 2] and res[1][1] == [1, 3]
    # every rank sees all 4 records, identical, ordered by block
    assert res[0][2] == res[1][2]
    metas = [BlockMeta.unpack(np.array(r)) for r in res[0][2]]
    assert [m.block for m in metas] == [0, 1, 2, 3]
    assert [m.rank for m in metas] == [0, 1, 0, 1]
    # records agree with a serial recomputation
    shape = (17, 17, 9)
    specs = split_blocks(shape, (2, 2, 1))
    field = oracle_mod.smooth_field(shape)
    for m in metas:
        s = specs[m.block]
        v = extract_block(field, shape, s)
        cls, L = oracle_mod.decompose(v, s.shape)
        off = oracle_mod.class_offsets(s.shape, L)
        parts = [cls[off[l]:off[l + 1]] for l in range(L + 1)]
        assert m.levels == L and m.shape == s.shape and m.origin == s.origin
        assert m.class_bytes == [p.size * 8 for p in parts]
        assert m.class_crc32 == class_crc32(parts)
