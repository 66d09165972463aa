"""Summarise an ncu --csv --metrics launch list: one line per launch."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = OrderedDict()
for r in rows[hi + 1:]:
    if len(r) > vi:
        d.setdefault((r[ii], r[ki]), {})[r[mi]] = r[vi]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for (i, k), v in list(d.items())[:n]:
    print(i, k.split("(")[0][:48], *(v.get(m, "") for m in sorted(v)))
print("metrics:", sorted(next(iter(d.values()))))
