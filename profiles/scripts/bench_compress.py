#!/usr/bin/env python3
"""Compression leg: mgr::compress / decompress of a
smooth field through the device path (FAST policy) next to the reference
(oracle/_ref, one host thread, smaller sample).  One JSON line.
  python profiles/scripts/bench_compress.py [--shape 513,513,513] [--eb 1e-4]"""
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
    ap.add_argument("--shape", default="513,513,513")
    ap.add_argument("--eb", type=float, default=1e-4)
    ap.add_argument("--ref-shape", default="129,129,129")
    a = ap.parse_args()
    import torch

    from bench import field_factors, make_field_device
    from paper_2105_12764_b200 import Plan

    shape = tuple(int(s) for s in a.shape.split(","))
    v = make_field_device(shape, 0, torch.device("cuda", 0), "float32")
    raw = v.numel() * 4
    out = {"component": "compress/decompress (SURVEY §8(f) row 2)", "shape": list(shape),
           "error_bound": a.eb, "raw_bytes": raw}
    plan = Plan(shape, "float32", fast=True)
    for codec, name in ((0, "store"), (1, "zlib")):
        plan.compress(v, a.eb, codec)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        data, b, m = plan.compress(v, a.eb, codec)
        tc = time.perf_counter() - t0
        t0 = time.perf_counter()
        back, *_ = plan.decompress(data)
        torch.cuda.synchronize()
        td = time.perf_counter() - t0
        err = float((back - v).abs().max())
        out[name] = {"compress_s": round(tc, 3), "compress_GBps": round(raw / tc / 1e9, 3),
                     "decompress_s": round(td, 3), "decompress_GBps": round(raw / td / 1e9, 3),
                     "ratio": round(raw / len(data), 2), "bin": b, "measured": m,
                     "roundtrip_max_err": err}
    try:
        import oracle

        rs = tuple(int(s) for s in a.ref_shape.split(","))
        fac = field_factors(rs, 0)
        vv = np.zeros(rs[::-1])
        for term, w in ((0, 1.0), (1, 0.6), (2, 0.2)):
            vv += w * np.einsum("k,j,i->kji", fac[2][term], fac[1][term], fac[0][term])
        vv = vv.astype(np.float32).reshape(-1)
        t0 = time.perf_counter()
        data, b, m = oracle.ref_compress(vv, rs, a.eb, 1)
        tc = time.perf_counter() - t0
        t0 = time.perf_counter()
        oracle.ref_decompress(data, vv.size, np.float32)
        td = time.perf_counter() - t0
        out["reference_cpu"] = {"shape": list(rs), "codec": "zlib", "cores": 1,
                                "compress_GBps": round(vv.nbytes / tc / 1e9, 4),
                                "decompress_GBps": round(vv.nbytes / td / 1e9, 4),
                                "ratio": round(vv.nbytes / len(data), 2)}
    except Exception as e:  # noqa: BLE001
        out["reference_cpu"] = {"error": str(e)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
