#!/usr/bin/env python3
"""Print the key metrics of an exported ncu raw CSV (profiles/scripts/ncu_one.sh)."""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(d.get("Kernel Name", "?")[:90])
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]} {units[hdr.index(k)]}")
        stalls = sorted(((float(d[k]) if d[k] not in ("", "n/a") else 0.0, k) for k in hdr
                         if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")),
                        reverse=True)[:8]
        tot = sum(float(d[k]) for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not k.endswith("not_issued") and d[k] not in ("", "n/a")) or 1
        for v, k in stalls:
            print(f"  stall {k[len('smsp__pcsamp_warps_issue_stalled_'):]:40s} {100*v/tot:.1f}%")
