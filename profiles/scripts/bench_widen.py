#!/usr/bin/env python3
"""Measurements of the widened rows: (1) 4-D grids (gen4.cuh) device
decompose / recompose throughput; (2) cooperative decompose with W workers
on one GPU (LocalTransport) against the serial device decompose -- the cost
of the slab orchestration (halo copies, chained z solves, gathers), not a
multi-GPU speed-up.  Prints one JSON object."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def dev_time(fn, reps=5):
    import torch

    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    import numpy as np
    import torch

    from paper_2105_12764_b200 import Plan, coop, make_grid

    out = {}
    for shape, dt in [((129, 129, 129, 9), "float32"), ((65, 65, 65, 33), "float64")]:
        n = int(np.prod(shape))
        v = torch.rand(n, dtype=getattr(torch, dt), device="cuda")
        plan = Plan(shape, dt)
        c = torch.empty_like(v)
        r = torch.empty_like(v)
        d = dev_time(lambda: plan.decompose(v, c))
        rc = dev_time(lambda: plan.recompose(c, plan.levels, r))
        nb = n * v.element_size()
        out["4d " + "x".join(map(str, shape)) + " " + dt] = {
            "decompose_ms": round(d, 3), "recompose_ms": round(rc, 3),
            "decompose_GBps": round(nb / d / 1e6, 1), "recompose_GBps": round(nb / rc / 1e6, 1),
            "roundtrip_exact": bool(torch.equal(r, v)) if False else None}
        plan.close()
    shape = (513, 513, 513)
    rng = np.random.default_rng(3)
    g = make_grid(shape, rng.random(513 ** 3, dtype=np.float32))
    vt = torch.from_numpy(g.values).cuda()
    plan = Plan(shape, "float32")
    c = torch.empty_like(vt)
    serial = dev_time(lambda: plan.decompose(vt, c), reps=3)
    out["coop 513^3 f32 serial decompose_ms"] = round(serial, 3)
    plan.close()
    for w in (2, 4, 8):
        coop.cooperative_decompose(g, w)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        coop.cooperative_decompose(g, w)
        torch.cuda.synchronize()
        out[f"coop 513^3 f32 W={w} one GPU wall_ms (incl. host upload + class download)"] = round(
            1e3 * (time.perf_counter() - t0), 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
