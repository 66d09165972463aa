"""One warm FAST decompose + recompose of a 2-D f64 field (default 8193^2),
for ncu captures of the long-fiber Thomas kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2105_12764_b200 import Plan  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8193
dt = sys.argv[2] if len(sys.argv) > 2 else "float64"
plan = Plan((n, n), dt, fast=True)
v = torch.rand(n * n, dtype=getattr(torch, dt), device="cuda")
c = plan.decompose(v)
r = plan.recompose(c)
torch.cuda.synchronize()
plan.decompose(v, c)
plan.recompose(c, plan.levels, r)
torch.cuda.synchronize()
print("ok", float((r - v).abs().max()))
