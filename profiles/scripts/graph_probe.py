#!/usr/bin/env python3
"""Eager launches vs one CUDA graph replay of decompose + full recompose
(1025^3 f32 FAST): how much of the step is launch overhead."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    import torch

    from bench import make_field_device
    from paper_2105_12764_b200 import Plan

    shape = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1025,1025,1025").split(","))
    dev = torch.device("cuda", 0)
    v = make_field_device(shape, 0, dev, "float32")
    plan = Plan(shape, "float32", fast=True)
    c = torch.empty_like(v)
    r = torch.empty_like(v)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            plan.decompose(v, c, s)
            plan.recompose(c, plan.levels, r, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 20
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(K):
            plan.decompose(v, c, s)
            plan.recompose(c, plan.levels, r, s)
        e1.record(s)
    torch.cuda.synchronize()
    print("eager ms/step", e0.elapsed_time(e1) / K)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.decompose(v, c, s)
        plan.recompose(c, plan.levels, r, s)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        g.replay()
        e0.record(s)
        for _ in range(K):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    print("graph ms/step", e0.elapsed_time(e1) / K)


if __name__ == "__main__":
    main()
