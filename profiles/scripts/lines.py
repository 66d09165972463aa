#!/usr/bin/env python3
"""Executed warp instructions per CUDA source line for one kernel of the
in-tree libmgrg.so, from an exported ncu SASS page (ncu_one.sh) and the
library's line table (nvdisasm -g):
  python profiles/scripts/lines.py gpurun_out/TAG.sass.csv.gz <mangled-kernel-name>"""
import collections
import csv
import gzip
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def line_map(name):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all",
                    os.path.join(ROOT, "paper_2105_12764_b200", "libmgrg.so")], cwd=d,
                   capture_output=True)
    cubin = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cubin)],
                         capture_output=True, text=True).stdout.split("\n")
    start = next(i for i, l in enumerate(txt) if l.startswith(name + ":"))
    out, cur = {}, None
    for l in txt[start:]:
        if l.strip().startswith(".section") and out:
            break
        m = re.search(r'## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
        m2 = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m2:
            out[int(m2.group(1), 16)] = cur
    return out


def main():
    path, name = sys.argv[1], sys.argv[2]
    mp = line_map(name)
    rows = list(csv.reader(io.TextIOWrapper(gzip.open(path), "utf-8")))
    hdr = rows[1]
    iA, iE = hdr.index("Address"), hdr.index("Instructions Executed")
    data = [(int(r[iA], 16), int(r[iE] or 0)) for r in rows[2:] if len(r) > iE]
    base = data[0][0]
    agg = collections.Counter()
    for a, n in data:
        agg[mp.get(a - base)] += n
    tot = sum(agg.values())
    srcs = {}
    for (k, n) in agg.most_common(40):
        if k is None:
            print(f"{100 * n / tot:5.1f}% ?")
            continue
        f, l = k
        p = os.path.join(ROOT, "paper_2105_12764_b200", "csrc", f)
        if p not in srcs:
            srcs[p] = open(p).read().split("\n") if os.path.exists(p) else []
        s = srcs[p][l - 1].strip()[:80] if len(srcs[p]) >= l else ""
        print(f"{100 * n / tot:5.1f}% {f}:{l} {s}")


if __name__ == "__main__":
    main()
