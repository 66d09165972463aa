"""One class_crc32 pass over a 1025^3 f32 class buffer (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2105_12764_b200 import Plan  # noqa: E402

plan = Plan((1025, 1025, 1025), "float32", fast=True)
c = torch.rand(plan.num_elements, device="cuda")
print(plan.class_crc32(c))
