#!/usr/bin/env python3
"""ncu-verified bandwidth of one decompose + one recompose: sum of
dram__bytes_read + dram__bytes_write over the library's kernels divided by the
sum of their durations (cold cache, serialised -- ncu's own replay), split at
the first recompose kernel.   python profiles/scripts/step_dram.py step_dram.csv [peak_GBps]"""
import collections
import csv
import json
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
         "usecond": 1e-6, "nsecond": 1e-9, "ms": 1e-3, "msecond": 1e-3}


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    hdr = rows[0]
    iid, ik, im, iu, iv = (hdr.index(x) for x in
                           ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        if "mgrg::" not in r[ik]:
            continue
        v = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
        per[int(r[iid])][r[im]] = v
        names[int(r[iid])] = r[ik]
    phase = "decompose"
    tot = {"decompose": [0.0, 0.0], "recompose": [0.0, 0.0]}
    for i in sorted(per):
        if "rload" in names[i] or "rgpk" in names[i]:
            phase = "recompose"
        d = per[i]
        tot[phase][0] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        tot[phase][1] += d.get("gpu__time_duration.sum", 0)
    peak = float(sys.argv[2]) if len(sys.argv) > 2 else None
    out = {}
    for k, (b, t) in tot.items():
        out[k] = {"dram_bytes": b, "kernel_s": t, "GBps": round(b / t / 1e9, 1)}
        if peak:
            out[k]["frac_of_peak"] = round(b / t / 1e9 / peak, 3)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
