#!/usr/bin/env python3
"""Summarise ncu captures (.ncu-rep, --set full) into the numbers the
roofline uses: duration, DRAM bytes, throughput, issue activity, and the
SASS instruction mix per fine element.  Runs offline (ncu -i).

  python profiles/ncu_summary.py OUT.md REP[:elements] ...
"""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, "--csv", *args], capture_output=True,
                         text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarise(rep, elements=None):
    rows = ncu_csv(rep, "--page", "raw")
    hdr, units = rows[0], rows[1]
    lines = []
    for row in rows[2:]:
        name = row[hdr.index("Kernel Name")]
        lines.append(f"### `{name[:110]}`\n")
        lines.append("| metric | value |\n|---|---|")
        for m, label in METRICS:
            if m in hdr:
                i = hdr.index(m)
                lines.append(f"| {label} (`{m}`) | {row[i]} {units[i]} |")
        if "dram__bytes_read.sum" in hdr:
            rd = float(row[hdr.index("dram__bytes_read.sum")])
            wr = float(row[hdr.index("dram__bytes_write.sum")])
            u = units[hdr.index("dram__bytes_read.sum")]
            scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}.get(u, 1)
            lines.append(f"| traffic read+write | {(rd + wr) * scale:.4e} B |")
        lines.append("")
    sass = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    h = sass[1]
    ii, si = h.index("Instructions Executed"), h.index("Source")
    c, tot = collections.Counter(), 0
    for row in sass[2:]:
        try:
            n = int(row[ii])
        except (ValueError, IndexError):
            continue
        t = row[si].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        c[op] += n
        tot += n
    if tot:
        per = f" (per element: {tot / elements:.2f})" if elements else ""
        lines.append(f"SASS warp instructions: {tot}{per}; top opcodes: " +
                     ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in c.most_common(12)))
        lines.append("")
    return "\n".join(lines)


def main():
    out = sys.argv[1]
    parts = ["# ncu summaries\n"]
    for arg in sys.argv[2:]:
        rep, _, el = arg.partition(":")
        parts.append(f"## {rep}\n")
        parts.append(summarise(rep, float(el) if el else None))
    open(out, "w").write("\n".join(parts))


if __name__ == "__main__":
    main()
