#!/usr/bin/env python3
"""PCIe budget of the e2e leg (1025^3 f32): pinned H2D / D2H alone and
concurrently, and decompose_host / recompose_host split."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    import torch

    from bench import make_field_device
    from paper_2105_12764_b200 import Plan

    shape = (1025, 1025, 1025)
    N = 1025 ** 3
    dev = torch.device("cuda", 0)
    d = make_field_device(shape, 0, dev, "float32")
    h1 = torch.empty(N, dtype=torch.float32, pin_memory=True)
    h2 = torch.empty(N, dtype=torch.float32, pin_memory=True)
    h3 = torch.empty(N, dtype=torch.float32, pin_memory=True)
    d2 = torch.empty_like(d)
    h1.copy_(d)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    gb = N * 4 / 1e9

    def t(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps

    h2d = t(lambda: d2.copy_(h1, non_blocking=True))
    d2h = t(lambda: h2.copy_(d, non_blocking=True))

    def both():
        with torch.cuda.stream(s1):
            d2.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d, non_blocking=True)
    bo = t(both)
    print(f"H2D {gb / h2d:.1f} GB/s  D2H {gb / d2h:.1f} GB/s  both {2 * gb / bo:.1f} GB/s aggregate "
          f"({bo * 1e3:.1f} ms for {gb:.2f} GB each way)")
    plan = Plan(shape, "float32", fast=True)
    hin, hcls, hout = h1.numpy(), h2.numpy(), h3.numpy()
    dec = t(lambda: plan.decompose_host(hin, hcls))
    rec = t(lambda: plan.recompose_host(hcls, plan.levels, hout))
    print(f"decompose_host {dec * 1e3:.1f} ms  recompose_host {rec * 1e3:.1f} ms  "
          f"e2e {2 * gb / (dec + rec):.1f} GB/s")


if __name__ == "__main__":
    main()
