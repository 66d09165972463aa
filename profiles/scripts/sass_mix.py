#!/usr/bin/env python3
"""Opcode mix (executed warp instructions) and top stall lines of an exported
ncu SASS source page (profiles/scripts/ncu_one.sh):
  python profiles/scripts/sass_mix.py gpurun_out/TAG.sass.csv.gz [elements]"""
import collections
import csv
import gzip
import io
import sys

path = sys.argv[1]
elems = float(sys.argv[2]) if len(sys.argv) > 2 else None
rows = list(csv.reader(io.TextIOWrapper(gzip.open(path), "utf-8")))
hdr = rows[1]
iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index(
    "Warp Stall Sampling (All Samples)")
mix = collections.Counter()
tot = 0
lines = []
for r in rows[2:]:
    if len(r) <= iE or not r[iE]:
        continue
    n = int(r[iE])
    op = r[iS].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1]
    o = o.split(".")[0]
    mix[o] += n
    tot += n
    lines.append((int(r[iW] or 0), r[0], r[iS].strip()))
print(f"total warp instructions {tot:.4e}" + (f"  per element {tot / elems:.3f}" if elems else ""))
for o, n in mix.most_common(25):
    print(f"  {o:10s} {100 * n / tot:5.1f}%" + (f"  {n / elems:.3f}/elem" if elems else ""))
print("top stall lines:")
for w, a, s in sorted(lines, reverse=True)[:25]:
    print(f"  {w:7d} {s}")
