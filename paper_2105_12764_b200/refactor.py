"""Python mirror of the reference's public refactoring API
(/root/reference/proj/include/mgr/refactor.hpp:18-76, 462-534 and
grid.hpp:19-55): same names, argument meaning and error behaviour, with the
work done by the CUDA path through the C ABI (plan.Plan).

Host (numpy) inputs go through the host entry points (H2D, device path,
D2H); torch CUDA tensors stay on the device."""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Any, Optional

import numpy as np

from . import errors
from .plan import Plan

kDefaultTileBudget = 32768  # kernels.hpp:31
kMaxDims = 4                # ndarray.hpp:12


def uniform_coords(n: int) -> np.ndarray:
    """grid.cpp:7-12."""
    return np.arange(n, dtype=np.float64) / (n - 1) if n > 1 else np.zeros(1)


def _validate_geometry(shape, coords, min_extent):
    """validate_grid_geometry (grid.cpp:14-36)."""
    if len(shape) == 0 or len(shape) > kMaxDims:
        raise errors.InvalidGrid(
            f"grid must have 1..{kMaxDims} dimensions, got {len(shape)}")
    if len(coords) != len(shape):
        raise errors.InvalidGrid("coordinate arrays do not match dimension count")
    for d, n in enumerate(shape):
        if n < min_extent:
            raise errors.InvalidGrid(
                f"dimension {d} has {n} nodes; need at least {min_extent}")
        c = np.asarray(coords[d], dtype=np.float64)
        if c.size != n:
            raise errors.InvalidGrid(f"coordinates of dimension {d} do not match its extent")
        bad = np.nonzero(~(c[:-1] < c[1:]))[0]
        if bad.size:
            raise errors.InvalidGrid(
                f"coordinates of dimension {d} are not strictly increasing at index {bad[0]}")


@dataclass
class TensorGrid:
    """grid.hpp:19-26: values on a tensor product of strictly increasing
    coordinates, row-major with dimension 0 fastest."""

    shape: tuple
    coords: list
    values: Any  # numpy array (host) or torch CUDA tensor (device)

    def ndims(self) -> int:
        return len(self.shape)

    def size(self) -> int:
        return int(np.prod(self.shape))


def make_grid(shape, values, coords=None, min_extent: int = 3) -> TensorGrid:
    """make_grid (grid.hpp:34-50)."""
    shape = tuple(int(s) for s in shape)
    if coords is None or len(coords) == 0:
        coords = [uniform_coords(n) for n in shape]
    coords = [np.asarray(c, dtype=np.float64) for c in coords]
    _validate_geometry(shape, coords, min_extent)
    n = int(np.prod(shape))
    size = values.numel() if hasattr(values, "numel") else np.asarray(values).size
    if size != n:
        raise errors.ShapeError(f"value count {size} does not match grid of {n} nodes")
    if not hasattr(values, "numel"):
        values = np.ascontiguousarray(values).reshape(-1)
    return TensorGrid(shape, coords, values)


def value_range(g: TensorGrid) -> float:
    """grid.hpp:52-55."""
    v = g.values
    if hasattr(v, "numel"):
        return float(v.max().item()) - float(v.min().item())
    return float(np.max(v)) - float(np.min(v))


@dataclass
class PhaseCounters:
    in_: int = 0
    out: int = 0

    def total(self) -> int:
        return self.in_ + self.out


@dataclass
class LevelPassStats:
    """refactor.hpp:48-65."""

    level: int = 0
    level_elements: int = 0
    coefficient: PhaseCounters = field(default_factory=PhaseCounters)
    fused_copy: PhaseCounters = field(default_factory=PhaseCounters)
    masstrans: list = field(default_factory=list)
    solve: list = field(default_factory=list)
    apply: PhaseCounters = field(default_factory=PhaseCounters)

    def total_passes(self) -> float:
        t = self.coefficient.total() + self.fused_copy.total() + self.apply.total()
        t += sum(c.total() for c in self.masstrans) + sum(c.total() for c in self.solve)
        return t / self.level_elements if self.level_elements else 0.0


@dataclass
class PassStats:
    levels: list = field(default_factory=list)  # finest first


@dataclass
class RefactorOptions:
    """refactor.hpp:71-76.  ``levels`` caps the depth (value-affecting); the
    CPU tile shape does not exist on the device (launch configuration is
    internal and never changes values) and is accepted and ignored."""

    levels: Optional[int] = None
    tile: Any = None
    tile_budget: int = kDefaultTileBudget
    stats: Optional[PassStats] = None
    device: int = 0


@dataclass
class RefactoredData:
    """refactor.hpp:18-32.  ``classes[l]`` are views into one flat buffer
    (``flat``), class l at offset N_{l-1}."""

    shape: tuple
    coords: list
    levels: int
    classes: list
    flat: Any = None

    def total_elements(self) -> int:
        return int(sum(len(c) if not hasattr(c, "numel") else c.numel()
                       for c in self.classes))


@dataclass
class ReconstructionReport:
    classes_used: int = 0
    max_abs_error: float = 0.0
    rel_linf_error: float = 0.0
    weighted_l2_error: float = 0.0
    elapsed_seconds: float = 0.0


_PLANS: dict = {}


def _plan_for(shape, coords, dtype, levels, device) -> Plan:
    """Plans are cached per geometry (hierarchy build + workspace allocation
    happen once, like a reusable engine)."""
    key = (tuple(shape), str(dtype), levels, device,
           None if coords is None else np.concatenate(
               [np.asarray(c, dtype=np.float64) for c in coords]).tobytes())
    p = _PLANS.get(key)
    if p is None:
        p = Plan(shape, dtype, coords=coords, levels=levels, device=device)
        _PLANS[key] = p
    return p


def _level_stats(plan: Plan, l: int) -> LevelPassStats:
    nd = len(plan.shape)
    ls, cs = plan.level_shape(l), plan.level_shape(l - 1)
    F, C = int(np.prod(ls)), int(np.prod(cs))
    lv = LevelPassStats(level=l, level_elements=F)
    lv.coefficient = PhaseCounters(F, F - C)
    lv.fused_copy = PhaseCounters(0, F - C)
    cur = F
    for d in range(nd):
        if cs[d] < ls[d]:
            out = cur // ls[d] * cs[d]
            lv.masstrans.append(PhaseCounters(cur, out))
            lv.solve.append(PhaseCounters(2 * C, 2 * C))
            cur = out
        else:
            lv.masstrans.append(PhaseCounters())
            lv.solve.append(PhaseCounters())
    lv.apply = PhaseCounters(2 * C, C)
    return lv


def _fill_stats(stats: PassStats, plan: Plan, recompose: bool = False):
    """The per-level traffic counters the reference engine accumulates
    (refactor.hpp:223-421): decompose clears and appends levels finest
    first; recompose appends levels coarsest first without clearing
    (refactor.hpp:159-199).  Acceptance criterion 9 (acceptance.cpp:336-374)
    checks this composition."""
    if not recompose:
        stats.levels.clear()
        stats.levels.extend(_level_stats(plan, l) for l in range(plan.levels, 0, -1))
    else:
        stats.levels.extend(_level_stats(plan, l) for l in range(1, plan.levels + 1))


def _is_torch(x) -> bool:
    return hasattr(x, "is_cuda")


def _on_plan_device(t, plan: Plan):
    if t.is_cuda and t.device.index == plan.device:
        return t.contiguous()
    return t.to(f"cuda:{plan.device}").contiguous()


def decompose(grid: TensorGrid, opt: RefactorOptions | None = None) -> RefactoredData:
    """mgr::decompose (refactor.hpp:462-474)."""
    opt = opt or RefactorOptions()
    _validate_geometry(grid.shape, grid.coords, 2)
    vals = grid.values
    dtype = vals.dtype
    plan = _plan_for(grid.shape, grid.coords if not _all_uniform(grid) else None,
                     dtype, opt.levels, opt.device)
    if _is_torch(vals):
        # a block handed to another GPU's worker moves to that GPU first
        flat = plan.decompose(_on_plan_device(vals.reshape(-1), plan))
    else:
        flat = plan.decompose_host(np.asarray(vals).reshape(-1))
    if opt.stats is not None:
        _fill_stats(opt.stats, plan)
    classes = [flat[s] for s in plan.class_slices()]
    return RefactoredData(tuple(grid.shape), [np.asarray(c) for c in grid.coords],
                          plan.levels, classes, flat)


def decompose_spatiotemporal(snapshots, time_coords,
                             opt: RefactorOptions | None = None) -> RefactoredData:
    """mgr::decompose_spatiotemporal (refactor.hpp:536-567): stack the
    snapshots along a trailing time dimension and decompose the stacked grid
    (spatial dimensions before the temporal one at every level).  A 3-D
    snapshot series becomes a 4-D grid (csrc/gen4.cuh)."""
    if len(snapshots) < 2:
        raise errors.ShapeError("need at least 2 snapshots")
    if len(time_coords) != len(snapshots):
        raise errors.ShapeError("time coordinate count does not match snapshots")
    first = snapshots[0]
    if first.ndims() + 1 > kMaxDims:
        raise errors.InvalidGrid("too many dimensions after stacking time")
    for s in snapshots:
        same = tuple(s.shape) == tuple(first.shape) and len(s.coords) == len(first.coords)
        same = same and all(np.array_equal(np.asarray(a, dtype=np.float64),
                                           np.asarray(b, dtype=np.float64))
                            for a, b in zip(s.coords, first.coords))
        if not same:
            raise errors.ShapeError("snapshots must share shape and coordinates")
    shape = tuple(first.shape) + (len(snapshots),)
    coords = [np.asarray(c, dtype=np.float64) for c in first.coords]
    coords.append(np.asarray(time_coords, dtype=np.float64))
    if _is_torch(first.values):
        import torch

        values = torch.cat([s.values.reshape(-1) for s in snapshots])
    else:
        values = np.concatenate([np.asarray(s.values).reshape(-1) for s in snapshots])
    stacked = make_grid(shape, values, coords, 2)
    return decompose(stacked, opt)


def _all_uniform(g) -> bool:
    for d, n in enumerate(g.shape):
        c = np.asarray(g.coords[d], dtype=np.float64)
        if not np.array_equal(c, uniform_coords(n)):
            return False
    return True


def _addr(a) -> int:
    return a.data_ptr() if _is_torch(a) else int(a.__array_interface__["data"][0])


def flat_if_current(r: RefactoredData, plan: Plan, upto: int | None = None):
    """r.flat when classes 0..upto are all still views of it at their class
    offsets (N_{l-1}) -- i.e. nobody replaced a class array (quantized,
    zeroed, loaded from elsewhere); None otherwise.  The reference treats
    the classes as the data (refactor.hpp:18-32), so a stale flat buffer
    must never be used in their place."""
    flat = r.flat
    if flat is None:
        return None
    upto = r.levels if upto is None else upto
    if len(r.classes) < upto + 1 or _is_torch(flat) != _is_torch(r.classes[0]):
        return None
    offs = plan.class_offsets
    es = flat.element_size() if _is_torch(flat) else flat.itemsize
    base = _addr(flat)
    for l in range(upto + 1):
        c = r.classes[l]
        n = c.numel() if _is_torch(c) else c.size
        if n != offs[l + 1] - offs[l] or (n and _addr(c) != base + offs[l] * es):
            return None
        if _is_torch(c) and (not c.is_contiguous() or c.dtype != flat.dtype):
            return None
        if not _is_torch(c) and (not c.flags.c_contiguous or c.dtype != flat.dtype):
            return None
    return flat


def _flat_classes(r: RefactoredData, k: int, plan: Plan):
    flat = flat_if_current(r, plan, k)
    if flat is not None:
        return flat
    parts = r.classes[: k + 1]
    if parts and _is_torch(parts[0]):
        import torch

        return torch.cat([p.reshape(-1) for p in parts])
    return np.concatenate([np.asarray(p).reshape(-1) for p in parts])


def recompose(r: RefactoredData, classes_used: int,
              opt: RefactorOptions | None = None) -> TensorGrid:
    """mgr::recompose (refactor.hpp:476-496)."""
    opt = opt or RefactorOptions()
    if classes_used > r.levels or classes_used < 0:
        raise errors.InvalidLevel(
            f"requested {classes_used} classes; container has {r.levels}")
    for l in range(classes_used + 1):
        if l >= len(r.classes):
            raise errors.MissingClass(f"class {l} not loaded")
    g0 = TensorGrid(tuple(r.shape), r.coords, None)
    first = r.classes[0]
    plan = _plan_for(r.shape, r.coords if not _all_uniform(g0) else None,
                     first.dtype, r.levels, opt.device)
    flat = _flat_classes(r, classes_used, plan)
    if _is_torch(flat):
        vals = plan.recompose(_on_plan_device(flat, plan), classes_used)
    else:
        vals = plan.recompose_host(np.asarray(flat), classes_used)
    if opt.stats is not None:
        _fill_stats(opt.stats, plan, recompose=True)
    return TensorGrid(tuple(r.shape), r.coords, vals)


def weighted_l2_norm(g: TensorGrid) -> float:
    """sqrt(v^T (M_0 x M_1 x ...) v) with the finest mass matrices, fp64
    (grid.hpp:198-244).  Reporting metric only (not on the refactoring
    path)."""
    v = g.values
    v = v.detach().cpu().numpy() if _is_torch(v) else np.asarray(v)
    w = v.astype(np.float64).reshape(tuple(reversed(g.shape)))
    for d in range(len(g.shape)):
        ax = len(g.shape) - 1 - d
        h = np.diff(np.asarray(g.coords[d], dtype=np.float64))
        x = np.moveaxis(w, ax, -1)
        out = np.empty_like(x)
        n = x.shape[-1]
        out[..., 0] = (2 * h[0]) * x[..., 0] + h[0] * x[..., 1]
        if n > 2:
            out[..., 1:-1] = (h[:-1] * x[..., :-2] + (2 * (h[:-1] + h[1:])) * x[..., 1:-1]
                              + h[1:] * x[..., 2:])
        out[..., -1] = h[-1] * x[..., -2] + (2 * h[-1]) * x[..., -1]
        w = np.moveaxis(out, -1, ax)
    dot = float(np.dot(w.reshape(-1), v.astype(np.float64).reshape(-1)))
    return float(np.sqrt(max(dot, 0.0)))


def recompose_with_report(r: RefactoredData, classes_used: int,
                          reference: TensorGrid | None = None,
                          opt: RefactorOptions | None = None):
    """refactor.hpp:500-534."""
    t0 = time.perf_counter()
    g = recompose(r, classes_used, opt)
    rep = ReconstructionReport(classes_used=classes_used)
    ref = reference
    if ref is None:
        best = min(r.levels, len(r.classes) - 1 if r.classes else 0)
        ref = g if classes_used == best else recompose(r, best, opt)

    def host(x):
        return x.detach().cpu().numpy() if _is_torch(x) else np.asarray(x)

    gv, rv = host(g.values).astype(np.float64), host(ref.values).astype(np.float64)
    diff = gv - rv
    rep.max_abs_error = float(np.max(np.abs(diff))) if diff.size else 0.0
    rng = float(rv.max() - rv.min())
    rep.rel_linf_error = rep.max_abs_error / rng if rng > 0 else rep.max_abs_error
    dt = host(g.values).dtype
    rep.weighted_l2_error = weighted_l2_norm(
        TensorGrid(g.shape, g.coords, diff.astype(dt)))
    rep.elapsed_seconds = time.perf_counter() - t0
    return g, rep
