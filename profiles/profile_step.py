#!/usr/bin/env python3
"""One decompose + one full recompose of a synthetic field on cuda:0 -- the
command the ncu captures under profiles/ were taken on (no warm-up, so the
launch order is: decompose levels L..1, then recompose levels 1..L).

  python profiles/profile_step.py [--shape 1025,1025,1025] [--dtype float32] [--fast]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="1025,1025,1025")
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--fast", action="store_true")
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    import torch

    from bench import make_field_device
    from paper_2105_12764_b200 import Plan

    shape = tuple(int(s) for s in a.shape.split(","))
    dev = torch.device("cuda", 0)
    v = make_field_device(shape, 0, dev, a.dtype) if len(shape) == 3 else \
        torch.rand(int(torch.tensor(shape).prod()), dtype=getattr(torch, a.dtype), device=dev)
    plan = Plan(shape, a.dtype, fast=a.fast)
    torch.cuda.synchronize()
    for _ in range(a.reps):
        c = plan.decompose(v)
        r = plan.recompose(c)
    torch.cuda.synchronize()
    print("levels", plan.levels, "roundtrip max err", (r - v).abs().max().item())


if __name__ == "__main__":
    main()
