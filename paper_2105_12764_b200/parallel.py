"""Block-sharded (embarrassingly parallel) refactoring across GPUs.

The reference's data-parallel mode is ``embarrassing_decompose``
(/root/reference/proj/include/mgr/parallel_impl.hpp:810-847, declared
parallel.hpp:243-247): independent blocks, a small worker pool, result i ==
``decompose(blocks[i])`` (test_parallel.cpp:216-223), the first failure
aborts with ``WorkerFailure``.  On B200 a worker is a GPU:

* :func:`embarrassing_decompose` / :func:`embarrassing_recompose` -- one
  process, one host thread per visible GPU, blocks claimed from a shared
  counter exactly like the reference's pool;
* :class:`BlockShardedRefactor` -- one process per GPU under
  ``torch.distributed`` (the production layout): blocks dealt round-robin to
  ranks, no data-path collective, ONE all-gather of fixed-size per-block
  metadata records at the end (NCCL over NVLink for CUDA tensors; gloo in the
  CPU tests).

:func:`split_blocks` / :func:`assemble_blocks` cut a large field into blocks
that share their boundary planes and put
recomposed blocks back together (shared planes from the lower block).
"""
from __future__ import annotations

import threading
import time
import zlib
from dataclasses import dataclass

import numpy as np

from . import errors
from .refactor import RefactoredData, RefactorOptions, TensorGrid

META_WORDS = 48       # int64 words per block metadata record
MAX_CLASSES = 32      # class count capacity of a record (L + 1 <= 32)


# ---------------------------------------------------------------------------
# block geometry
# ---------------------------------------------------------------------------
@dataclass
class BlockSpec:
    """One block of a larger field: global origin and extents per dimension
    (dimension 0 fastest)."""

    index: int
    origin: tuple
    shape: tuple


def split_points(n: int, parts: int) -> list:
    """Boundary node indices of `parts` blocks along an extent-n dimension;
    neighbouring blocks share the boundary node.  For n - 1 divisible by
    parts the blocks are equal (2049 / 2 -> [0, 1024, 2048])."""
    if parts < 1 or n - 1 < parts:
        raise errors.InvalidGrid(f"cannot split {n} nodes into {parts} blocks")
    return [((n - 1) * k) // parts for k in range(parts + 1)]


def split_blocks(shape, parts) -> list:
    """Blocks of a `shape` field cut `parts[d]` ways along dimension d,
    sharing boundary planes; block index runs dimension 0 fastest (block b
    of a 2x2x2 split has b_x = b & 1, b_y = (b >> 1) & 1, b_z = b >> 2)."""
    shape = tuple(int(s) for s in shape)
    parts = tuple(int(p) for p in parts)
    if len(parts) != len(shape):
        raise errors.ShapeError("one split count per dimension")
    pts = [split_points(n, p) for n, p in zip(shape, parts)]
    out = []
    counts = [len(p) - 1 for p in pts]
    total = int(np.prod(counts))
    for b in range(total):
        idx, r = [], b
        for c in counts:
            idx.append(r % c)
            r //= c
        origin = tuple(pts[d][i] for d, i in enumerate(idx))
        ext = tuple(pts[d][i + 1] - pts[d][i] + 1 for d, i in enumerate(idx))
        out.append(BlockSpec(b, origin, ext))
    return out


def _slices(spec: BlockSpec):
    # numpy arrays of the field are indexed [..., z, y, x] (dim 0 fastest)
    return tuple(slice(o, o + s) for o, s in zip(reversed(spec.origin), reversed(spec.shape)))


def extract_block(values: np.ndarray, shape, spec: BlockSpec) -> np.ndarray:
    """Copy of one block's values (flat, dimension 0 fastest)."""
    v = np.asarray(values).reshape(tuple(reversed(tuple(shape))))
    return np.ascontiguousarray(v[_slices(spec)]).reshape(-1)


def block_grid(values: np.ndarray, shape, coords, spec: BlockSpec) -> TensorGrid:
    """TensorGrid of one block; coordinates are the global slices."""
    c = [np.asarray(coords[d], dtype=np.float64)[o:o + s]
         for d, (o, s) in enumerate(zip(spec.origin, spec.shape))]
    return TensorGrid(tuple(spec.shape), c, extract_block(values, shape, spec))


def assemble_blocks(block_values, specs, shape, dtype=None) -> np.ndarray:
    """Inverse of split_blocks: shared boundary planes are taken from the
    lower block (blocks written in descending index order, so the lowest
    block touching a plane writes it last)."""
    shape = tuple(int(s) for s in shape)
    dtype = dtype or np.asarray(block_values[0]).dtype
    out = np.empty(tuple(reversed(shape)), dtype=dtype)
    for spec in sorted(specs, key=lambda s: -s.index):
        bv = block_values[spec.index]
        if hasattr(bv, "detach"):
            bv = bv.detach().cpu().numpy()
        out[_slices(spec)] = np.asarray(bv).reshape(tuple(reversed(spec.shape)))
    return out.reshape(-1)


def assign_blocks(nblocks: int, rank: int, world: int) -> list:
    """Round-robin dealing of blocks to ranks (grouped_decompose's dealing,
    parallel_impl.hpp:849-885): rank r gets r, r + world, ..."""
    if world < 1 or not 0 <= rank < world:
        raise errors.TooManyWorkers(f"rank {rank} outside world of {world}")
    return list(range(rank, nblocks, world))


# ---------------------------------------------------------------------------
# metadata records (the only cross-GPU exchange)
# ---------------------------------------------------------------------------
@dataclass
class BlockMeta:
    block: int
    rank: int
    origin: tuple
    shape: tuple
    dtype_bytes: int
    levels: int
    class_bytes: list     # byte length of every class 0..L
    class_crc32: list     # crc32 of every class payload (pipeline.cpp:13-28 polynomial)
    decompose_us: int = 0
    recompose_us: int = 0
    checksum: int = 0     # crc32 of the class CRCs (filled by block_meta)

    def pack(self) -> np.ndarray:
        if self.levels + 1 > MAX_CLASSES // 2:
            raise errors.Unsupported("too many classes for a metadata record")
        r = np.zeros(META_WORDS, dtype=np.int64)
        r[0], r[1] = self.block, self.rank
        r[2:2 + len(self.origin)] = self.origin
        r[6:6 + len(self.shape)] = self.shape
        r[10], r[11] = len(self.shape), self.dtype_bytes
        r[12], r[13], r[14] = self.levels, self.decompose_us, self.recompose_us
        n = self.levels + 1
        r[15:15 + n] = self.class_bytes
        r[31:31 + n] = self.class_crc32
        return r

    @staticmethod
    def unpack(r) -> "BlockMeta":
        r = [int(x) for x in r]
        nd, L = r[10], r[12]
        return BlockMeta(block=r[0], rank=r[1], origin=tuple(r[2:2 + nd]),
                         shape=tuple(r[6:6 + nd]), dtype_bytes=r[11], levels=L,
                         class_bytes=r[15:16 + L], class_crc32=r[31:32 + L],
                         decompose_us=r[13], recompose_us=r[14])


def class_crc32(classes) -> list:
    """CRC-32 (zlib polynomial, as the MGRF container, pipeline.cpp:13-28) of
    every class payload."""
    out = []
    for c in classes:
        if hasattr(c, "detach"):
            c = c.detach().cpu().numpy()
        out.append(zlib.crc32(np.ascontiguousarray(c).view(np.uint8)) & 0xFFFFFFFF)
    return out


def gather_metadata(records, max_blocks_per_rank: int, group=None, device=None):
    """All-gather of every rank's fixed-size metadata records (one
    collective, microseconds).  `records`: this rank's BlockMeta list.
    Returns every rank's records ordered by block index."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    buf = np.full((max_blocks_per_rank, META_WORDS), -1, dtype=np.int64)
    for i, m in enumerate(records):
        buf[i] = m.pack()
    t = torch.from_numpy(buf.reshape(-1))
    if device is not None:
        t = t.to(device)
    out = torch.empty(world * t.numel(), dtype=torch.int64, device=t.device)
    dist.all_gather_into_tensor(out, t, group=group)
    allr = out.cpu().numpy().reshape(world * max_blocks_per_rank, META_WORDS)
    metas = [BlockMeta.unpack(r) for r in allr if r[0] >= 0]
    return sorted(metas, key=lambda m: m.block)


# ---------------------------------------------------------------------------
# the native gather: libmgrg's NCCL communicator (include/mgrg.h mgrg_comm_*)
# ---------------------------------------------------------------------------
def _to_c(m: BlockMeta):
    from . import _lib

    c = _lib.BlockMeta()
    c.block_id, c.rank, c.dtype = m.block, m.rank, m.dtype_bytes
    c.ndims, c.levels = len(m.shape), m.levels
    for d in range(len(m.shape)):
        c.origin[d], c.shape[d] = int(m.origin[d]), int(m.shape[d])
    for l in range(m.levels + 1):
        c.class_bytes[l] = int(m.class_bytes[l])
        c.class_crc32[l] = int(m.class_crc32[l]) & 0xFFFFFFFF
    c.decompose_ms, c.recompose_ms = m.decompose_us / 1e3, m.recompose_us / 1e3
    return c


def _from_c(c) -> BlockMeta:
    nd, L = int(c.ndims), int(c.levels)
    return BlockMeta(block=int(c.block_id), rank=int(c.rank), origin=tuple(c.origin[:nd]),
                     shape=tuple(c.shape[:nd]), dtype_bytes=int(c.dtype), levels=L,
                     class_bytes=list(c.class_bytes[:L + 1]),
                     class_crc32=list(c.class_crc32[:L + 1]),
                     decompose_us=int(round(c.decompose_ms * 1e3)),
                     recompose_us=int(round(c.recompose_ms * 1e3)))


def block_meta(plan, d_classes, block: int, rank: int, origin=None,
               decompose_ms: float = 0.0, recompose_ms: float = 0.0,
               stream=None) -> BlockMeta:
    """The block's metadata record from the device class buffer:
    mgrg_block_meta_fill (per-class CRC-32 on the GPU, geometry from the
    plan)."""
    import ctypes

    from . import _lib
    from .plan import _stream_ptr, _tensor_ptr

    c = _lib.BlockMeta()
    org = None
    if origin is not None:
        org = (ctypes.c_uint64 * 4)(*[int(x) for x in origin])
    _lib.check(_lib.lib().mgrg_block_meta_fill(
        plan._h, _tensor_ptr(d_classes), int(block), int(rank), org,
        float(decompose_ms), float(recompose_ms), ctypes.byref(c),
        _stream_ptr(stream, plan.device)))
    m = _from_c(c)
    m.checksum = int(c.checksum)
    return m


class NativeMetaComm:
    """One NCCL communicator per rank inside libmgrg (mgrg_comm_init), for
    the block-sharded path's one collective: the metadata all-gather
    (mgrg_comm_allgather_block_meta).  The 128-byte unique id made by rank 0
    is shipped to the other ranks through the process group's own
    transport."""

    def __init__(self, rank: int, world: int, device: int, uid: bytes):
        import ctypes

        from . import _lib

        self.rank, self.world, self.device = int(rank), int(world), int(device)
        self._h = ctypes.c_void_p()
        buf = (ctypes.c_uint8 * _lib.MGRG_COMM_ID_BYTES).from_buffer_copy(uid)
        _lib.check(_lib.lib().mgrg_comm_init(buf, self.world, self.rank, self.device,
                                             ctypes.byref(self._h)))

    @staticmethod
    def unique_id() -> bytes:
        import ctypes

        from . import _lib

        buf = (ctypes.c_uint8 * _lib.MGRG_COMM_ID_BYTES)()
        _lib.check(_lib.lib().mgrg_comm_unique_id(buf))
        return bytes(buf)

    @classmethod
    def from_process_group(cls, group=None, device: int | None = None):
        import torch
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0)
                                   if group is not None else 0, group=group)
        dev = torch.cuda.current_device() if device is None else int(device)
        return cls(rank, world, dev, obj[0])

    def allgather(self, records, per_rank: int):
        """Every rank's records (this rank's `records`, padded to per_rank),
        ordered by block index."""
        from . import _lib

        mine = (_lib.BlockMeta * max(1, per_rank))()
        for i in range(per_rank):
            mine[i].block_id = -1
        for i, m in enumerate(records):
            mine[i] = _to_c(m)
        out = (_lib.BlockMeta * max(1, per_rank * self.world))()
        _lib.check(_lib.lib().mgrg_comm_allgather_block_meta(self._h, mine, int(per_rank),
                                                             out, None))
        metas = [_from_c(out[i]) for i in range(per_rank * self.world)
                 if out[i].block_id >= 0]
        return sorted(metas, key=lambda m: m.block)

    def close(self):
        from . import _lib

        if self._h:
            _lib.lib().mgrg_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# single-process pool: one host thread per GPU
# ---------------------------------------------------------------------------
def _pool(n_items: int, workers: int, fn):
    import torch

    if not torch.cuda.is_available():
        raise errors.CudaError("no CUDA device: the refactoring path has no CPU fallback")
    ndev = torch.cuda.device_count()
    pool = max(1, min(int(workers), n_items, ndev))
    out = [None] * n_items
    lock = threading.Lock()
    state = {"next": 0, "err": None}

    def run(dev):
        torch.cuda.set_device(dev)
        while True:
            with lock:
                i = state["next"]
                state["next"] += 1
                if i >= n_items or state["err"] is not None:
                    return
            try:
                out[i] = fn(i, dev)
            except Exception as e:  # first failure stops the pool
                with lock:
                    if state["err"] is None:
                        state["err"] = e
                return

    ths = [threading.Thread(target=run, args=(d,)) for d in range(pool)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if state["err"] is not None:
        raise errors.WorkerFailure(str(state["err"]))
    return out


def embarrassing_decompose(blocks, workers: int, opt: RefactorOptions | None = None):
    """parallel_impl.hpp:810-847 with GPUs as workers: result i equals
    ``decompose(blocks[i])`` bit-for-bit; pass counters are not filled
    (``o.stats = nullptr``, :830-831)."""
    from .refactor import decompose

    if not blocks:
        return []
    base = opt or RefactorOptions()

    def one(i, dev):
        o = RefactorOptions(levels=base.levels, tile=base.tile,
                            tile_budget=base.tile_budget, stats=None, device=dev)
        return decompose(blocks[i], o)

    return _pool(len(blocks), workers, one)


def embarrassing_recompose(results, classes_used, workers: int,
                           opt: RefactorOptions | None = None):
    """Per-block recompose on the same pool (the reference has no parallel
    recompose driver; this mirrors embarrassing_decompose)."""
    from .refactor import recompose

    base = opt or RefactorOptions()

    def one(i, dev):
        k = classes_used if classes_used is not None else results[i].levels
        return recompose(results[i], k, RefactorOptions(levels=base.levels, device=dev))

    return _pool(len(results), workers, one)


# ---------------------------------------------------------------------------
# one process per GPU (torch.distributed)
# ---------------------------------------------------------------------------
class BlockShardedRefactor:
    """Blocks dealt round-robin to the ranks of a process group, each rank
    refactoring its blocks on its own GPU with no data-path communication;
    ``finish()`` all-gathers the per-block metadata (the one collective)."""

    def __init__(self, nblocks: int, group=None, device=None):
        import torch.distributed as dist

        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.nblocks = int(nblocks)
        self.mine = assign_blocks(self.nblocks, self.rank, self.world)
        self.max_per_rank = -(-self.nblocks // self.world)
        self.device = device
        self.records: list = []

    def record(self, block: int, spec_or_shape, result: RefactoredData, dtype_bytes: int,
               decompose_s: float = 0.0, recompose_s: float = 0.0, crc: bool = True):
        if isinstance(spec_or_shape, BlockSpec):
            origin, shape = spec_or_shape.origin, spec_or_shape.shape
        else:
            origin, shape = (0,) * len(spec_or_shape), tuple(spec_or_shape)
        sizes = [int(c.numel() if hasattr(c, "numel") else np.asarray(c).size) * dtype_bytes
                 for c in result.classes]
        m = BlockMeta(block=block, rank=self.rank, origin=tuple(origin), shape=tuple(shape),
                      dtype_bytes=dtype_bytes, levels=result.levels, class_bytes=sizes,
                      class_crc32=class_crc32(result.classes) if crc else [0] * len(sizes),
                      decompose_us=int(decompose_s * 1e6), recompose_us=int(recompose_s * 1e6))
        self.records.append(m)
        return m

    def decompose_local(self, make_grid_for_block, opt: RefactorOptions | None = None,
                        crc: bool = True):
        """Decompose every block this rank owns; make_grid_for_block(i) ->
        (TensorGrid, BlockSpec|shape).  Returns {block: RefactoredData}."""
        import torch

        from .refactor import decompose

        out = {}
        for i in self.mine:
            g, spec = make_grid_for_block(i)
            t0 = time.perf_counter()
            r = decompose(g, opt)
            if torch.cuda.is_available():
                torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            esize = np.dtype(str(r.classes[0].dtype).replace("torch.", "")).itemsize
            self.record(i, spec, r, esize, decompose_s=dt, crc=crc)
            out[i] = r
        return out

    def finish(self, comm: "NativeMetaComm | None" = None):
        """The metadata all-gather: every rank learns every block's record --
        through libmgrg's own NCCL communicator when one is given (the C-ABI
        path a C++ caller uses), else through the process group (gloo in the
        CPU tests)."""
        if comm is not None:
            return comm.allgather(self.records, self.max_per_rank)
        return gather_metadata(self.records, self.max_per_rank, self.group, self.device)
