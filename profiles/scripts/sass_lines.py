#!/usr/bin/env python3
"""Executed warp instructions per CUDA source line: joins an ncu SASS source
page export (profiles/scripts/ncu_one.sh: TAG.sass.csv.gz, absolute
addresses + executed counts) with nvdisasm --print-line-info of the same
kernel in the shipped cubin (offsets -> file:line).
  python profiles/scripts/sass_lines.py TAG.sass.csv.gz all.sass MANGLED [top]"""
import collections
import csv
import gzip
import io
import re
import sys

sass_csv, dis, fn = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rows = list(csv.reader(io.TextIOWrapper(gzip.open(sass_csv), "utf-8")))
hdr = rows[1]
iA, iS, iE = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
iW = hdr.index("Warp Stall Sampling (All Samples)")
recs = [(int(r[iA], 16), r[iS].strip(), float(r[iE] or 0), float(r[iW] or 0)) for r in rows[2:]]
base = recs[0][0]
# offset -> (file:line)
lines = {}
cur = None
inside = False
for ln in open(dis):
    if ln.startswith(f".text.{fn}:"):
        inside = True
        continue
    if inside and ln.startswith(".text.") :
        break
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
    if m:
        lines[int(m.group(1), 16)] = cur
by_line = collections.Counter()
stall = collections.Counter()
ops = collections.defaultdict(collections.Counter)
tot = sum(e for _, _, e, _ in recs)
for a, s, e, w in recs:
    key = lines.get(a - base, "?")
    by_line[key] += e
    stall[key] += w
    op = s.split()[0] if not s.startswith("@") else s.split()[1]
    ops[key][op.split(".")[0]] += e
print(f"total {tot:.4e}")
for key, e in by_line.most_common(top):
    mix = ", ".join(f"{o} {100 * c / e:.0f}" for o, c in ops[key].most_common(4))
    print(f"{100 * e / tot:5.1f}%  stall {stall[key]:7.0f}  {key:22s} {mix}")
