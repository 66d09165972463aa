#!/usr/bin/env python3
"""Markdown summary of exported ncu captures (raw CSV + SASS page) and of an
ncu launch list (gpu__time_duration per launch):
  python profiles/scripts/summarize.py OUT.md --launches L.csv TAG=raw.csv[:sass.csv.gz[:elements]] ..."""
import collections
import csv
import gzip
import io
import sys

KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("smsp__inst_executed.sum", "warp instructions"),
        ("launch__registers_per_thread", "registers/thread"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 throughput %"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %")]


def raw_section(tag, path, sass=None, elems=None):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        out.append(f"### {tag}: `{d.get('Kernel Name', '?')[:100]}`\n")
        out.append("| metric | value |\n|---|---|")
        for k, lab in KEYS:
            if k in d:
                out.append(f"| {lab} (`{k}`) | {d[k]} {units[hdr.index(k)]} |")
        st = [(float(d[k]), k) for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not k.endswith("not_issued") and d[k] not in ("", "n/a")]
        tot = sum(v for v, _ in st) or 1
        top = ", ".join(f"{k.split('stalled_')[1]} {100 * v / tot:.0f}%"
                        for v, k in sorted(st, reverse=True)[:6])
        out.append(f"\nstall samples: {top}\n")
    if sass:
        rows = list(csv.reader(io.TextIOWrapper(gzip.open(sass), "utf-8")))
        h = rows[1]
        iS, iE = h.index("Source"), h.index("Instructions Executed")
        mix = collections.Counter()
        for r in rows[2:]:
            if len(r) > iE and r[iE]:
                op = r[iS].strip().split()
                if not op:
                    continue
                o = op[1] if op[0].startswith("@") else op[0]
                mix[o.split(".")[0]] += int(r[iE])
        tot = sum(mix.values())
        per = f" ({tot / elems:.2f} per fine element)" if elems else ""
        out.append(f"SASS warp instructions {tot:.3e}{per}; top opcodes: " +
                   ", ".join(f"{o} {100 * n / tot:.1f}%" for o, n in mix.most_common(12)) + "\n")
    return "\n".join(out)


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    iN, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    g = collections.Counter()
    n = collections.Counter()
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    for r in rows[1:]:
        k = r[iN].split("(")[0].replace("void ", "")
        if not k.startswith("mgrg::"):
            continue  # torch kernels of the harness (field generation, checks)
        g[k] += float(r[iV].replace(",", "")) * scale.get(r[iU], 1.0)
        n[k] += 1
    tot = sum(g.values())
    out = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, v in g.most_common():
        out.append(f"| `{k[:70]}` | {n[k]} | {v:.1f} | {100 * v / tot:.1f}% |")
    return "\n".join(out)


def main():
    outp = sys.argv[1]
    args = sys.argv[2:]
    parts = ["# ncu summaries\n"]
    if args and args[0] == "--launches":
        parts.append("## Launch list (ncu --metrics gpu__time_duration.sum, cold cache, "
                     "serialised; mgrg kernels only, share of their sum)\n\n" +
                     launches(args[1]) + "\n")
        args = args[2:]
    parts.append("## Full captures (--set full)\n")
    for a in args:
        tag, rest = a.split("=", 1)
        f = rest.split(":")
        parts.append(raw_section(tag, f[0], f[1] if len(f) > 1 else None,
                                 float(f[2]) if len(f) > 2 else None))
    open(outp, "w").write("\n".join(parts) + "\n")


if __name__ == "__main__":
    main()
