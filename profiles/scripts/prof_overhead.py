#!/usr/bin/env python3
"""Step time of 1025^3 f32 FAST dec + rec with per-launch profiling events on
the top 2 levels / the top level / none (the bench's timed region records
the top 2): do the events cost step time?"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    import torch

    from bench import make_field_device
    from paper_2105_12764_b200 import Plan

    shape = (1025, 1025, 1025)
    dev = torch.device("cuda", 0)
    v = make_field_device(shape, 0, dev, "float32")
    p = Plan(shape, "float32", fast=True)
    c, r = torch.empty_like(v), torch.empty_like(v)
    s = torch.cuda.current_stream()
    out = {}
    for rep in range(2):
        for mode in ("top2", "top1", "none"):
            if mode == "none":
                p.set_profiling(False)
            else:
                p.set_profiling(True, top_levels=2 if mode == "top2" else 1)
            for _ in range(3):
                p.decompose(v, c, s)
                p.recompose(c, p.levels, r, s)
            torch.cuda.synchronize()
            p.profile(reset=True) if mode != "none" else None
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(40):
                p.decompose(v, c, s)
                p.recompose(c, p.levels, r, s)
            e1.record(s)
            torch.cuda.synchronize()
            out[f"{mode}_{rep}"] = round(e0.elapsed_time(e1) / 40, 4)
            if mode != "none":
                p.profile(reset=True)
    print(json.dumps({"ms_per_step": out}))


if __name__ == "__main__":
    main()
