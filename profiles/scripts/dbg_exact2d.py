#!/usr/bin/env python3
"""Localise an exact-policy mismatch: decompose classes vs the oracle for a
few 2-D shapes / seeds, and the unit kernels (gpk, masstrans, solve) on every
level of the failing ones."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402


def main():
    import torch

    from paper_2105_12764_b200 import Plan

    for shape in [(100, 37), (100, 36), (99, 37), (37, 100), (64, 37), (100, 9, 5)]:
        for dt in ("float32", "float64"):
            for nonuni in (False, True):
                for seed in range(3):
                    rng = np.random.default_rng(seed)
                    coords = ([np.cumsum(rng.uniform(0.1, 1.0, n)) for n in shape]
                              if nonuni else None)
                    v = rng.random(int(np.prod(shape))).astype(dt)
                    plan = Plan(shape, dt, coords=coords)
                    got = plan.decompose(torch.from_numpy(v).cuda()).cpu().numpy()
                    ref, L = oracle.decompose(v, shape, coords)
                    bad = [l for l, s in enumerate(plan.class_slices())
                           if not np.array_equal(got[s], ref[s])]
                    if bad:
                        print("MISMATCH", shape, dt, nonuni, seed, "classes", bad,
                              "max", float(np.abs(got.astype(np.float64) - ref).max()))
                        # unit kernels per level
                        nd = len(shape)
                        for l in range(1, L + 1):
                            ls = tuple(int(x) for x in plan.level_shape(l))
                            cs = tuple(int(x) for x in plan.level_shape(l - 1))
                            F, C = int(np.prod(ls)), int(np.prod(cs))
                            x = rng.standard_normal(F).astype(dt)
                            d = torch.from_numpy(x.copy()).cuda()
                            plan.gpk(l, d)
                            ok_g = np.array_equal(d.cpu().numpy(), oracle.gpk(x, shape, l, False, coords=coords))
                            oks = []
                            for dim in range(nd):
                                ie = [cs[k] if k < dim else ls[k] for k in range(nd)]
                                oe = list(ie)
                                oe[dim] = cs[dim]
                                y = rng.standard_normal(int(np.prod(ie))).astype(dt)
                                ro, _ = oracle.masstrans(y, shape, l, dim, int(np.prod(oe)),
                                                         fused_copy=False, class_size=F - C,
                                                         coords=coords)
                                o = torch.empty(int(np.prod(oe)), dtype=getattr(torch, dt), device="cuda")
                                plan.masstrans(l, dim, torch.from_numpy(y).cuda(), o)
                                oks.append(("mt", dim, bool(np.array_equal(o.cpu().numpy(), ro))))
                                z = rng.standard_normal(C).astype(dt)
                                dz = torch.from_numpy(z.copy()).cuda()
                                plan.solve(l, dim, dz)
                                oks.append(("solve", dim, bool(np.array_equal(dz.cpu().numpy(), oracle.solve(z, shape, l, dim, coords=coords)))))
                            print("   level", l, ls, "gpk", ok_g, oks)
                    plan.close()
    print("done")


if __name__ == "__main__":
    main()
