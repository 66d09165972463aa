#!/usr/bin/env python3
"""Per-class FAST-policy error vs the CPU oracle (range-normalized), for
debugging kernel changes on the GPU box:  python profiles/scripts/check_fast.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    import torch

    import oracle
    from paper_2105_12764_b200 import Plan

    shapes = [(3, 3, 3), (5, 9, 17), (65, 33, 129), (33, 17, 257), (97, 65, 33),
              (257, 257), (9, 5), (129, 9, 65)]
    rng = np.random.default_rng(7)
    bad = 0
    for dt in ("float32", "float64"):
        for shape in shapes:
            for nonuni in (False, True):
                coords = ([np.cumsum(rng.uniform(0.1, 1.0, n)) for n in shape]
                          if nonuni else None)
                v = rng.random(int(np.prod(shape))).astype(dt)
                rv = float(v.max() - v.min())
                plan = Plan(shape, dt, coords=coords, fast=True)
                ref, L = oracle.decompose(v, shape, coords)
                got = plan.decompose(torch.from_numpy(v).cuda()).cpu().numpy()
                errs = []
                for s in plan.class_slices():
                    errs.append(float(np.abs(got[s].astype(np.float64) - ref[s]).max() / rv)
                                if s.stop > s.start else 0.0)
                back = plan.recompose(torch.from_numpy(got).cuda()).cpu().numpy()
                rt = float(np.abs(back.astype(np.float64) - v).max() / rv)
                tol = 1e-5 if dt == "float32" else 1e-12
                ok = max(errs) <= tol and rt <= tol
                bad += not ok
                print(f"{'ok ' if ok else 'BAD'} {dt} {shape} nonuni={nonuni} L={L} "
                      f"class_err={['%.1e' % e for e in errs]} rt={rt:.1e}", flush=True)
                plan.close()
    print("bad", bad)


if __name__ == "__main__":
    main()
