"""Device time of the GPU CRC-32 (CUDA events): all 11 class records of a
1025^3 f32 class buffer (mgrg_class_crc32) and one 4.3 GB range
(mgrg_crc32), checked against zlib on a 64 MiB prefix."""
import json
import os
import sys
import zlib

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2105_12764_b200 import Plan, crc32  # noqa: E402

plan = Plan((1025, 1025, 1025), "float32", fast=True)
c = torch.rand(plan.num_elements, device="cuda")
nbytes = plan.num_elements * 4
out = {"bytes": nbytes}
for name, fn in (("class_crc32_all", lambda: plan.class_crc32(c)), ("crc32_one_range", lambda: crc32(c))):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):  # per call: each call ends in a host sync (CRCs to the host)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    out[name] = {"ms_median": round(ms, 3), "ms_min": round(ts[0], 3), "ms_max": round(ts[-1], 3),
                 "GBps_median": round(nbytes / ms / 1e6, 1)}
pre = c[: (64 << 20) // 4]
out["zlib_match_64MiB"] = crc32(pre) == zlib.crc32(pre.cpu().numpy().tobytes())
for a, b in ((0, 12345677), (0, 12345805), (3, 12345805), (1, 200), (0, 128 * 64 + 128)):
    x = c[a:b]
    out[f"zlib_match_{a}_{b}"] = crc32(x) == zlib.crc32(x.cpu().numpy().tobytes())
print(json.dumps(out))
