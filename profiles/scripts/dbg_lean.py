import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import oracle
from paper_2105_12764_b200 import Plan
shape = tuple(int(x) for x in sys.argv[1].split(","))
v = (np.arange(int(np.prod(shape))) % 7).astype("float64") ** 2
plan = Plan(shape, "float64", fast=True)
got = plan.decompose(torch.from_numpy(v).cuda()).cpu().numpy()
ref, L = oracle.decompose(v, shape, None)
np.set_printoptions(linewidth=200, precision=4, suppress=True)
print("offsets", plan.class_offsets)
print("got", got)
print("ref", ref)
print("diff idx", np.nonzero(np.abs(got - ref) > 1e-9)[0])
