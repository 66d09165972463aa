"""Cooperative multi-GPU decompose: one grid, several
GPUs, classes bit-identical to a serial decompose of the whole grid.

Mirrors mgr::cooperative_decompose (parallel.hpp:227-230,
parallel_impl.hpp:691-808) and make_partitions / split_dims_of
(parallel.cpp:9-90).  The reference runs worker threads over halo'd boxes
with a mailbox; here every worker is a GPU holding a plan for the WHOLE grid
(the 180 GB HBM makes full-size address spaces cheap) and owning a z slab of
every level lattice:

  level l, worker r owns coarse planes [c_r, c_{r+1}) (the last one through
  the top plane):
    halo    : fine planes 2c_r-2, 2c_r-1 from worker r-1, 2c_{r+1} from r+1
    level   : mgrg_coop_level -- coefficients, class-l stores of fine planes
              [2c_r, 2c_{r+1}), packed coarse values, load vector and its x/y
              solves (the serial kernels on a z range / sub-lattice)
    z solve : forward elimination chained r = 0..W-1, back substitution +
              apply chained r = W-1..0, carries = one xy plane, pipelined over
              fiber batches so W workers overlap (the reference's pipelined
              Thomas, parallel_impl.hpp:461-547)
  After the cooperative levels the (8^q times smaller) level lattice is
  gathered on worker 0, which decomposes the remaining levels with a plan
  for that lattice; the class fragments are gathered on worker 0.

Slab boundaries sit on multiples of 2^q level-L planes so every cooperative
level splits on coarse planes; q is as deep as the extent and worker count
allow.  Grids the cooperative kernels do not cover (not 3-D, even extents,
a non-refining dimension) are decomposed on worker 0 alone -- still the
serial result.

Transport: `LocalTransport` runs all workers in this process on one device
(copies between their buffers) -- the single-GPU test vehicle;
`DistTransport` runs one worker per torch.distributed rank (NCCL send/recv
between GPUs over NVLink/NVSwitch).  The device work is identical."""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib, errors
from .plan import Plan, _stream_ptr, _tensor_ptr


class PartitionScheme(enum.Enum):
    block = 0
    shifted_round_robin = 1


@dataclass
class Partition:
    """parallel.hpp:22-27: one worker-owned box [lo, hi) of the grid."""
    worker: int = 0
    lo: tuple = ()
    hi: tuple = ()
    block_coord: tuple = (0, 0)


def split_dims_of(shape, scheme: PartitionScheme, workers: int) -> list:
    """parallel.cpp:9-19."""
    nd = len(shape)
    if workers == 1:
        return []
    if scheme == PartitionScheme.block:
        return [nd - 1]
    if nd < 2:
        raise errors.ShapeError("shifted round-robin partitioning needs >= 2 dimensions")
    return [nd - 2, nd - 1]


def _split_range(n: int, parts: int) -> list:
    """Near-equal contiguous ranges, remainder to the leading ones
    (parallel.cpp:23-35)."""
    base, rem = divmod(n, parts)
    out, at = [], 0
    for i in range(parts):
        ln = base + (1 if i < rem else 0)
        out.append((at, at + ln))
        at += ln
    return out


def make_partitions(shape, workers: int, scheme: PartitionScheme) -> list:
    """make_partitions (parallel.cpp:37-90): block = slabs of the slowest
    dimension; shifted round-robin = workers^2 boxes over the two slowest
    dimensions, box (a, b) owned by worker (a + b) mod workers."""
    shape = tuple(int(s) for s in shape)
    if workers < 1:
        raise errors.TooManyWorkers("worker count must be positive")
    nd = len(shape)
    if workers == 1:
        return [Partition(0, (0,) * nd, shape, (0, 0))]
    split = split_dims_of(shape, scheme, workers)
    for d in split:
        if workers > shape[d]:
            raise errors.TooManyWorkers(
                f"cannot split dimension {d} of extent {shape[d]} across {workers} workers")
    parts = []
    if scheme == PartitionScheme.block:
        for w, (a, b) in enumerate(_split_range(shape[split[0]], workers)):
            lo, hi = [0] * nd, list(shape)
            lo[split[0]], hi[split[0]] = a, b
            parts.append(Partition(w, tuple(lo), tuple(hi), (w, 0)))
    else:
        ra = _split_range(shape[split[0]], workers)
        rb = _split_range(shape[split[1]], workers)
        for a in range(workers):
            for b in range(workers):
                lo, hi = [0] * nd, list(shape)
                lo[split[0]], hi[split[0]] = ra[a]
                lo[split[1]], hi[split[1]] = rb[b]
                parts.append(Partition((a + b) % workers, tuple(lo), tuple(hi), (a, b)))
    return parts


@dataclass
class CoopOptions:
    """parallel.hpp:61-71 (fault_injector: called at every phase entry as
    (worker, phase, level); an exception aborts the run as WorkerFailure)."""
    levels: Optional[int] = None
    scheme: PartitionScheme = PartitionScheme.block
    report: Optional["CommReport"] = None
    fault_injector: Optional[object] = None
    fast: bool = False
    batches: int = 8  # z-solve pipeline depth (fiber batches)


@dataclass
class CommPhaseStats:
    messages: int = 0
    elements: int = 0
    local_elements: int = 0
    seconds: float = 0.0


@dataclass
class CommReport:
    """parallel.hpp:36-58: per-phase message/element counts."""
    workers: int = 0
    scheme: PartitionScheme = PartitionScheme.block
    phases: dict = field(default_factory=dict)
    total_grid_elements: int = 0

    def add(self, phase: str, elements: int, remote: bool):
        st = self.phases.setdefault(phase, CommPhaseStats())
        st.messages += 1
        if remote:
            st.elements += elements
        else:
            st.local_elements += elements


# ---- slab geometry (host logic, CPU-tested) ---------------------------------
def coop_levels(level_shapes, workers: int) -> int:
    """Number q of cooperative (top) levels: slab boundaries on multiples of
    2^q level-L planes, every worker owning at least one 2^q unit, every
    cooperative level 3-D with odd extents refining in all dimensions."""
    L = len(level_shapes) - 1
    n2 = level_shapes[L][2] if len(level_shapes[L]) == 3 else 0
    if len(level_shapes[L]) != 3 or n2 < 3:
        return 0
    q = 0
    while q < L:
        nq = q + 1
        if (n2 - 1) % (1 << nq) or (n2 - 1) >> nq < workers:
            break
        l = L - q  # level that becomes cooperative
        ls, cs = level_shapes[l], level_shapes[l - 1]
        if any(n % 2 == 0 for n in ls) or any(c >= n for c, n in zip(cs, ls)):
            break
        q = nq
    return q


def slab_bounds(n2: int, workers: int, q: int) -> list:
    """Level-L plane boundaries B_0 = 0 < B_1 < ... < B_W = n2 - 1, multiples
    of 2^q (units dealt like _split_range)."""
    units = (n2 - 1) >> q
    return [a << q for a, _ in _split_range(units, workers)] + [n2 - 1]


def coarse_range(bounds, r: int, j: int, m2: int):
    """Worker r's coarse planes at cooperative level L - j."""
    c0 = bounds[r] >> (j + 1)
    c1 = m2 if r == len(bounds) - 2 else bounds[r + 1] >> (j + 1)
    return c0, c1


def class_layout3(ls):
    """make_class_layout (grid.cpp:140-165) of a 3-D level: (base, ext) per
    mask 1..7."""
    base, ext, off = {}, {}, 0
    for mask in range(1, 8):
        e = []
        for d in range(3):
            n = ls[d]
            ce = n // 2 + 1
            e.append(n - ce if (mask >> d) & 1 else ce)
        base[mask], ext[mask] = off, e
        off += e[0] * e[1] * e[2]
    return base, ext


def class_pieces(ls, c0: int, c1: int, m2: int):
    """(offset within class l, length) of the class-l fragments written by the
    worker owning coarse planes [c0, c1) (fine planes [2c0, 2c1)): per class
    type, z-major rows of its z ranks."""
    base, ext = class_layout3(ls)
    out = []
    for mask in range(1, 8):
        e = ext[mask]
        S = e[0] * e[1]
        if mask & 4:  # odd z planes 2zr+1 < n2 - 1
            a, b = min(c0, m2 - 1), min(c1, m2 - 1)
        else:
            a, b = c0, c1
        if b > a and S:
            out.append((base[mask] + S * a, S * (b - a)))
    return out


# ---- transports --------------------------------------------------------------
class LocalTransport:
    """All workers in this process (one device): messages are copies."""

    def __init__(self, workers: int):
        self.workers = workers
        self.local = list(range(workers))

    def move(self, pairs, report=None, phase=""):
        for src_r, src, dst_r, dst in pairs:
            dst.copy_(src)
            if report is not None:
                report.add(phase, src.numel(), src_r != dst_r)


class DistTransport:
    """One worker per torch.distributed rank: NCCL send/recv."""

    def __init__(self):
        import torch.distributed as dist

        self.dist = dist
        self.workers = dist.get_world_size()
        self.local = [dist.get_rank()]

    def move(self, pairs, report=None, phase=""):
        import torch

        dist = self.dist
        me = self.local[0]
        # gloo carries host tensors only: stage device buffers through the host
        # (NCCL moves device memory directly over NVLink)
        host = dist.get_backend() == "gloo"
        ops, post = [], []
        for src_r, src, dst_r, dst in pairs:
            if src_r == me and dst_r == me:
                dst.copy_(src)
            elif src_r == me:
                t = src.contiguous()
                ops.append(dist.P2POp(dist.isend, t.cpu() if host and t.is_cuda else t, dst_r))
            elif dst_r == me:
                if host and dst.is_cuda:
                    tmp = torch.empty(dst.shape, dtype=dst.dtype)
                    post.append((tmp, dst))
                    ops.append(dist.P2POp(dist.irecv, tmp, src_r))
                else:
                    ops.append(dist.P2POp(dist.irecv, dst, src_r))
            if report is not None and (src_r == me or dst_r == me):
                report.add(phase, (src if src_r == me else dst).numel(), src_r != dst_r)
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        for tmp, dst in post:
            dst.copy_(tmp)


# ---- the cooperative run -----------------------------------------------------
class _CudaView:
    """Zero-copy tensor over a plan-owned device buffer."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (ptr, False), "version": 2}


class _Worker:
    def __init__(self, rank, shape, dtype, coords, levels, device, fast):
        import torch

        self.rank = rank
        self.device = torch.device("cuda", device)
        self.plan = Plan(shape, dtype, coords=coords, levels=levels, device=device, fast=fast)
        self.tdt = getattr(torch, str(np.dtype(dtype)))
        N = int(np.prod(shape))
        self.inp = torch.zeros(N, dtype=self.tdt, device=self.device)
        self.cls = torch.zeros(N, dtype=self.tdt, device=self.device)

    def level_buf(self, level: int):
        import torch

        p = ctypes.c_void_p()
        _lib.check(_lib.lib().mgrg_plan_level_buffer(self.plan._h, level, ctypes.byref(p)))
        n = int(np.prod(self.plan.level_shape(level)))
        ts = "<f4" if self.tdt == torch.float32 else "<f8"
        return torch.as_tensor(_CudaView(p.value, n, ts), device=self.device)

    def level_array(self, level: int):
        """The packed level-`level` array (finest: the input buffer)."""
        L = self.plan.levels
        if level == L:
            return self.inp
        if level == 0:
            return self.cls[: int(np.prod(self.plan.level_shape(0)))]
        return self.level_buf(level)


def _fault(opt, w, phase, level):
    if opt.fault_injector is not None:
        try:
            opt.fault_injector(w, phase, level)
        except Exception as ex:  # parallel_impl.hpp:725-743
            raise errors.WorkerFailure(f"worker {w} failed in {phase}: {ex}") from ex


_FAULT_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int32, ctypes.c_char_p,
                             ctypes.c_int32)


def _native_cooperative(grid, workers, opt, device):
    """mgrg_cooperative_decompose_host: the same steps driven by the native
    runtime (csrc/coop_host.cuh), worker w on device (device + w) mod the
    visible GPUs."""
    from .plan import Plan
    from .refactor import RefactoredData

    shape = tuple(int(s) for s in grid.shape)
    vals = grid.values
    host = vals.detach().cpu().numpy() if hasattr(vals, "detach") else np.asarray(vals)
    host = np.ascontiguousarray(host.reshape(-1))
    coords = [np.asarray(c, dtype=np.float64) for c in grid.coords]
    desc = _lib.GridDesc()
    desc.ndims = len(shape)
    desc.dtype = host.dtype.itemsize
    for i, n in enumerate(shape):
        desc.shape[i] = n
    flat_c = np.ascontiguousarray(np.concatenate(coords))
    desc.coords = flat_c.ctypes.data
    desc.levels = int(opt.levels or 0)
    desc.device = device
    desc.flags = 1 if opt.fast else 0
    err = []

    def hook(ctx, w, phase, level):
        try:
            opt.fault_injector(int(w), phase.decode(), int(level))
            return 0
        except Exception as ex:  # surfaces as WorkerFailure
            err.append(ex)
            return 1

    cb = _FAULT_FN(hook) if opt.fault_injector is not None else None
    out = np.empty_like(host)
    moved = ctypes.c_uint64(0)
    _lib.check(_lib.lib().mgrg_cooperative_decompose_host(
        ctypes.byref(desc), workers, host.ctypes.data, out.ctypes.data,
        ctypes.cast(cb, ctypes.c_void_p) if cb else None, None, ctypes.byref(moved)))
    if opt.report is not None:
        opt.report.add("native", int(moved.value), True)
    plan = Plan(shape, host.dtype, coords=coords, levels=opt.levels, device=device)
    classes = [out[x] for x in plan.class_slices()]
    L = plan.levels
    plan.close()
    return RefactoredData(shape, coords, L, classes, out)


def cooperative_decompose(grid, workers: int, opt: CoopOptions | None = None,
                          transport=None, device: int = 0):
    """mgr::cooperative_decompose (parallel_impl.hpp:691-808).  Returns the
    RefactoredData on worker 0 (None on the other ranks).  Without a
    transport: the native runtime (mgrg_cooperative_decompose_host) drives
    all `workers` from this thread, worker w on device (device + w) mod the
    visible GPUs; LocalTransport(W): the same in Python on one device;
    DistTransport: one worker per rank (call on every rank)."""
    import torch

    from .refactor import RefactoredData, _validate_geometry

    opt = opt or CoopOptions()
    _validate_geometry(grid.shape, grid.coords, 2)
    make_partitions(grid.shape, workers, opt.scheme)  # reference validation
    if transport is None:
        if opt.report is not None:
            opt.report.workers, opt.report.scheme = workers, opt.scheme
            opt.report.total_grid_elements = int(np.prod(grid.shape))
        return _native_cooperative(grid, workers, opt, device)
    tp = transport
    if tp.workers != workers:
        raise errors.TooManyWorkers(f"transport has {tp.workers} workers, asked for {workers}")
    shape = tuple(int(s) for s in grid.shape)
    dtype = np.dtype(str(grid.values.dtype).replace("torch.", ""))
    coords = [np.asarray(c, dtype=np.float64) for c in grid.coords]
    if opt.report is not None:
        opt.report.workers, opt.report.scheme = workers, opt.scheme
        opt.report.total_grid_elements = int(np.prod(shape))
    ws = {r: _Worker(r, shape, dtype, coords, opt.levels,
                     device if transport is None else torch.cuda.current_device(), opt.fast)
          for r in tp.local}
    any_w = next(iter(ws.values()))
    plan0 = any_w.plan
    L = plan0.levels
    lshape = [tuple(int(x) for x in plan0.level_shape(l)) for l in range(L + 1)]
    q = coop_levels(lshape, workers) if workers > 1 else 0
    vals = grid.values
    host = vals.detach().cpu().numpy() if hasattr(vals, "detach") else np.asarray(vals)
    host = np.ascontiguousarray(host.reshape(-1), dtype=dtype)
    rep = opt.report
    s = torch.cuda.current_stream(any_w.device)

    if q == 0:
        # nothing to split on coarse planes: worker 0 decomposes alone
        if 0 in ws:
            _fault(opt, 0, "serial", L)
            w0 = ws[0]
            w0.inp.copy_(torch.from_numpy(host))
            w0.plan.decompose(w0.inp, w0.cls)
    else:
        n0, n1, n2 = lshape[L]
        nxy = n0 * n1
        bounds = slab_bounds(n2, workers, q)
        # upload: fine planes [2c0-2, 2c1] of level L
        for r, w in ws.items():
            c0, c1 = coarse_range(bounds, r, 0, lshape[L - 1][2])
            a, b = max(2 * c0 - 2, 0), min(2 * c1 + 1, n2)
            w.inp[a * nxy:b * nxy].copy_(torch.from_numpy(host[a * nxy:b * nxy]))
        for j in range(q):
            l = L - j
            ls, cs = lshape[l], lshape[l - 1]
            m0, m1, m2 = cs
            lxy, m01 = ls[0] * ls[1], m0 * m1
            rng = [coarse_range(bounds, r, j, m2) for r in range(workers)]
            if j > 0:  # halo planes of the level-l array
                arr = {r: w.level_array(l) for r, w in ws.items()}
                pairs = []
                for r in range(1, workers):
                    c0 = rng[r][0]
                    lo, hi = (2 * c0 - 2) * lxy, 2 * c0 * lxy
                    pairs.append((r - 1, arr[r - 1][lo:hi] if r - 1 in ws else None,
                                  r, arr[r][lo:hi] if r in ws else None))
                    lo, hi = 2 * c0 * lxy, (2 * c0 + 1) * lxy
                    pairs.append((r, arr[r][lo:hi] if r in ws else None,
                                  r - 1, arr[r - 1][lo:hi] if r - 1 in ws else None))
                tp.move(pairs, rep, "halo")
            for r, w in ws.items():
                _fault(opt, r, "level", l)
                c0, c1 = rng[r]
                _lib.check(_lib.lib().mgrg_coop_level(
                    w.plan._h, l, c0, c1, _tensor_ptr(w.inp) if l == L else None,
                    _tensor_ptr(w.cls), _stream_ptr(s)))
            # pipelined z solve: forward chain up, back substitution down
            B = max(1, min(opt.batches, m01)) if transport is not None else 1
            fb = [(m01 * b // B, m01 * (b + 1) // B) for b in range(B)]
            carry = {r: (torch.empty(m01, dtype=w.tdt, device=w.device),
                         torch.empty(m01, dtype=w.tdt, device=w.device)) for r, w in ws.items()}
            for direction in (0, 1):
                order = range(workers) if direction == 0 else range(workers - 1, -1, -1)
                order = list(order)
                for stage in range(workers + B - 1):
                    for pos, r in enumerate(order):
                        b = stage - pos
                        if not (0 <= b < B):
                            continue
                        f0, f1 = fb[b]
                        prev = order[pos - 1] if pos > 0 else None
                        if prev is not None:
                            src = carry[prev][1][f0:f1] if prev in ws else None
                            dst = carry[r][0][f0:f1] if r in ws else None
                            tp.move([(prev, src, r, dst)], rep, "solve")
                        if r in ws:
                            _fault(opt, r, "solve", l)
                            w = ws[r]
                            c0, c1 = rng[r]
                            _lib.check(_lib.lib().mgrg_coop_thomas_z(
                                w.plan._h, l, c0, c1, f0, f1, direction,
                                _tensor_ptr(carry[r][0]) if prev is not None else None,
                                _tensor_ptr(carry[r][1]), _tensor_ptr(w.cls), _stream_ptr(s)))
        # gather the level-(L-q) lattice on worker 0 and finish there
        lq = L - q
        ls = lshape[lq]
        lxy = ls[0] * ls[1]
        arr = {r: w.level_array(lq) for r, w in ws.items()}
        pairs = []
        for r in range(1, workers):
            c0, c1 = coarse_range(bounds, r, q - 1, ls[2])
            pairs.append((r, arr[r][c0 * lxy:c1 * lxy] if r in ws else None,
                          0, arr[0][c0 * lxy:c1 * lxy] if 0 in ws else None))
        tp.move(pairs, rep, "gather")
        if 0 in ws and lq >= 1:
            _fault(opt, 0, "tail", lq)
            w0 = ws[0]
            sub = Plan(ls, dtype, coords=_level_coords(coords, lshape, L, lq), levels=lq,
                       device=w0.device.index, fast=opt.fast)
            assert sub.levels == lq
            out = torch.empty(int(np.prod(ls)), dtype=w0.tdt, device=w0.device)
            sub.decompose(arr[0].clone(), out)
            w0.cls[: out.numel()].copy_(out)
            sub.close()
        # class fragments of the cooperative levels
        offs = plan0.class_offsets
        pairs = []
        for j in range(q):
            l = L - j
            m2 = lshape[l - 1][2]
            for r in range(1, workers):
                c0, c1 = coarse_range(bounds, r, j, m2)
                for o, n in class_pieces(lshape[l], c0, c1, m2):
                    a = int(offs[l]) + o
                    pairs.append((r, ws[r].cls[a:a + n] if r in ws else None,
                                  0, ws[0].cls[a:a + n] if 0 in ws else None))
        tp.move(pairs, rep, "classes")
    if 0 not in ws:
        return None
    w0 = ws[0]
    flat = w0.cls.cpu().numpy()
    sl = plan0.class_slices()
    classes = [flat[x] for x in sl]
    for w in ws.values():
        w.plan.close()
    return RefactoredData(shape, coords, L, classes, flat)


def _level_coords(coords, lshape, L, l):
    """Coordinates of the level-l lattice: positions {0, 2, 4, ..} + last,
    applied L - l times (grid.cpp:40-58)."""
    out = []
    for d, c in enumerate(coords):
        idx = np.arange(len(c))
        for _ in range(L - l):
            nxt = idx[::2]
            if nxt[-1] != idx[-1]:
                nxt = np.append(nxt, idx[-1])
            idx = nxt
        assert len(idx) == lshape[l][d]
        out.append(np.asarray(c, dtype=np.float64)[idx])
    return out


def grouped_decompose(blocks, num_groups: int, group_size: int,
                      scheme: PartitionScheme = PartitionScheme.block, devices=None):
    """mgr::grouped_decompose (parallel_impl.hpp:849-885): K groups of S
    cooperating workers; block i goes to group i mod K (round-robin) and
    result i == cooperative_decompose(blocks[i], S).  Group g runs on device
    g mod len(devices) (default: every visible GPU); the first failure
    surfaces as WorkerFailure."""
    import torch

    if num_groups < 1 or group_size < 1:
        raise errors.TooManyWorkers("group shape must be positive")
    groups = max(1, min(num_groups, len(blocks)))
    devs = list(devices) if devices else list(range(max(1, torch.cuda.device_count())))
    out = [None] * len(blocks)
    for i, b in enumerate(blocks):
        g = i % groups
        try:
            out[i] = cooperative_decompose(b, group_size, CoopOptions(scheme=scheme),
                                           device=devs[g % len(devs)])
        except errors.WorkerFailure:
            raise
        except Exception as ex:
            raise errors.WorkerFailure(str(ex)) from ex
    return out
