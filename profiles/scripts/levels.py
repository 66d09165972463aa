#!/usr/bin/env python3
"""Per-launch device times (CUDA events on the launch stream) of one warm
decompose + full recompose, grouped by kernel and level, with algorithmic
GB/s:  python profiles/scripts/levels.py [--shape 1025,1025,1025] [--exact]"""
import argparse
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="1025,1025,1025")
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--exact", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import torch

    from bench import make_field_device
    from paper_2105_12764_b200 import Plan

    shape = tuple(int(s) for s in a.shape.split(","))
    dev = torch.device("cuda", 0)
    v = (make_field_device(shape, 0, dev, a.dtype) if len(shape) == 3 else
         torch.rand(int(torch.tensor(shape).prod()), dtype=getattr(torch, a.dtype), device=dev))
    plan = Plan(shape, a.dtype, fast=not a.exact)
    c = plan.decompose(v)
    r = plan.recompose(c)
    torch.cuda.synchronize()
    plan.set_profiling(True)
    for _ in range(a.reps):
        plan.decompose(v, c)
        plan.recompose(c, plan.levels, r)
    torch.cuda.synchronize()
    prof = plan.profile(reset=True)
    g = collections.OrderedDict()
    for k, l, ms, by in prof:
        e = g.setdefault((k, l), [0.0, 0, by])
        e[0] += ms
        e[1] += 1
    tot = sum(e[0] for e in g.values()) / a.reps
    print(f"device total per dec+rec: {tot:.3f} ms")
    for (k, l), (ms, n, by) in g.items():
        t = ms / n
        print(f"  {k:12s} L{l:<2d} {t * 1e3:9.1f} us  {by / t / 1e6:8.1f} GB/s  x{n // a.reps}")


if __name__ == "__main__":
    main()
