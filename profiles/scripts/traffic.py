#!/usr/bin/env python3
"""Write profiles/ncu_traffic.json: dram__bytes_read.sum + dram__bytes_write.sum
per launch of the captured level kernels (exported ncu raw CSVs), keyed like
bench.py's per-kernel groups, "<kind>/L<level>/<arith>".
  python profiles/scripts/traffic.py KEY=path/to.raw.csv ..."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def traffic(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    r = rows[2]
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(m)
        tot += float(r[i]) * SCALE[units[i]]
    return int(tot)


def main():
    out_p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    out = json.load(open(out_p)) if os.path.exists(out_p) else {}
    for a in sys.argv[1:]:
        k, p = a.split("=", 1)
        out[k] = traffic(p)
    json.dump(out, open(out_p, "w"), indent=1, sort_keys=True)
    print(json.dumps(out, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
