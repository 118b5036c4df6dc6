#!/usr/bin/env python
"""Summarise ncu reports (run here, no GPU): key raw metrics + top stall
reasons per kernel, as JSON lines. usage: ncu_summary.py REP.ncu-rep [...]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "lts__t_bytes.sum", "launch__waves_per_multiprocessor"]


def summarize(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"report": path.split("/")[-1], "kernel": v[h.index("Kernel Name")]}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                d[k] = f"{v[i]} {units[i]}".strip()
        stalls = []
        for i, n in enumerate(h):
            if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued"):
                try:
                    stalls.append((float(v[i]), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        d["top_stalls_pct"] = {n: round(100 * s / tot, 1) for s, n in sorted(stalls, reverse=True)[:6]}
        res.append(d)
    return res


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for d in summarize(p):
            print(json.dumps(d))
