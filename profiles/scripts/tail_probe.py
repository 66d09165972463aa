#!/usr/bin/env python3
"""Cost of the small-level tail of the 1025^3 step: a (2^k+1)^3 f32 plan runs
exactly levels k..1 of the 1025^3 hierarchy (same extents), so its dec + rec
time with the bench's launch mode is the tail's device cost.  CUDA events,
100 warm iterations, PDL stream launches vs CUDA-graph replay."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2105_12764_b200 import Plan

    out = {}
    for n in (65, 129, 257, 513):
        shape = (n, n, n)
        v = torch.rand(n ** 3, device="cuda")
        for graphs in (False, True):
            p = Plan(shape, "float32", fast=True)
            c = torch.empty_like(v)
            r = torch.empty_like(v)
            s = torch.cuda.current_stream()
            p.set_graphs(graphs)
            for _ in range(5):
                p.decompose(v, c, s)
                p.recompose(c, p.levels, r, s)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(100):
                p.decompose(v, c, s)
                p.recompose(c, p.levels, r, s)
            e1.record(s)
            torch.cuda.synchronize()
            out[f"{n}^3 L{p.levels} {'graphs' if graphs else 'pdl'}"] = round(e0.elapsed_time(e1) / 100 * 1000, 1)
            p.close()
    print(json.dumps({"dec_plus_rec_us": out}))


if __name__ == "__main__":
    main()
