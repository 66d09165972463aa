#!/usr/bin/env python3
"""MGRF container leg at 1025^3 f32 (FAST decompose):
GPU CRC-32 of the class buffer (device GB/s against the HBM roofline), and the
write / prefix-read of the container through the device path (file system
bound), next to the reference writer (oracle/_ref, one host thread) on a
257^3 sample.  One JSON line.
  python profiles/scripts/bench_container.py [--dir /tmp]"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dir", default="/tmp")
    ap.add_argument("--shape", default="1025,1025,1025")
    a = ap.parse_args()
    import torch

    from bench import hbm_peak, make_field_device
    from paper_2105_12764_b200 import Plan, container

    shape = tuple(int(s) for s in a.shape.split(","))
    dev = torch.device("cuda", 0)
    v = make_field_device(shape, 0, dev, "float32")
    plan = Plan(shape, "float32", fast=True)
    c = plan.decompose(v)
    torch.cuda.synchronize()
    nbytes = c.numel() * 4
    # GPU CRC of the whole class buffer (all L+1 records)
    plan.class_crc32(c)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        crcs = plan.class_crc32(c)
    e1.record()
    torch.cuda.synchronize()
    crc_ms = e0.elapsed_time(e1) / reps
    peak, _ = hbm_peak()
    path = os.path.join(a.dir, "bench_container.mgrf")
    t0 = time.perf_counter()
    written = plan.write_refactored(c, path)
    t_w = time.perf_counter() - t0
    os.sync() if hasattr(os, "sync") else None
    out = torch.empty_like(c)
    t0 = time.perf_counter()
    _, loaded, used = plan.read_refactored(path, None, out)
    t_r = time.perf_counter() - t0
    k = plan.levels // 2
    t0 = time.perf_counter()
    _, _, used_k = plan.read_refactored(path, k, out)
    t_rk = time.perf_counter() - t0
    ok = bool(torch.equal(out[: plan.class_offsets[k + 1]], c[: plan.class_offsets[k + 1]]))
    os.remove(path)
    # reference writer on a bounded sample (one host thread, as the reference)
    ref = None
    try:
        import oracle

        if oracle.available("ref"):
            sn = (257, 257, 257)
            vs = np.random.default_rng(1).random(int(np.prod(sn))).astype(np.float32)
            cs, L = oracle.decompose(vs, sn, impl="ref")
            p2 = os.path.join(a.dir, "bench_container_ref.mgrf")
            t0 = time.perf_counter()
            nb = oracle.ref_write_refactored(cs, sn, L, p2)
            dt = time.perf_counter() - t0
            t0 = time.perf_counter()
            oracle.ref_read_refactored(p2, cs.size, np.float32)
            dr = time.perf_counter() - t0
            os.remove(p2)
            ref = {"sample": "257^3 f32 classes", "write_GBps": round(nb / dt / 1e9, 3),
                   "read_GBps": round(nb / dr / 1e9, 3), "cores": 1, "kind": "reference"}
    except Exception as e:  # noqa: BLE001
        ref = {"error": str(e)}
    print(json.dumps({
        "component": "MGRF container (SURVEY §8(f) row 1)", "shape": list(shape),
        "classes_bytes": nbytes, "levels": plan.levels,
        "crc32": {"ms": round(crc_ms, 3), "GBps": round(nbytes / crc_ms / 1e6, 1),
                  "roofline_frac_hbm_read": round(nbytes / crc_ms / 1e6 / peak, 3),
                  "records": len(crcs)},
        "write": {"bytes": written, "s": round(t_w, 3), "GBps": round(written / t_w / 1e9, 3),
                  "dir": a.dir},
        "read_all": {"bytes": used, "s": round(t_r, 3), "GBps": round(used / t_r / 1e9, 3)},
        "read_prefix": {"classes": k, "bytes": used_k, "s": round(t_rk, 3), "exact": ok},
        "reference_cpu": ref,
    }), flush=True)


if __name__ == "__main__":
    main()
