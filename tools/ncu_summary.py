#!/usr/bin/env python3
"""Compact summary of one ncu capture from its raw page.
    ncu -i X.ncu-rep --page raw --csv | python tools/ncu_summary.py "title"      (or: ... X_raw.csv[.gz] "title")
Prints duration, instruction count, issue-slot use, every execution-pipe
utilisation (IMAD / IMAD.WIDE run on the fma pipe), shared-memory bank
conflicts, L2 and DRAM bytes and throughput, and the stall reasons per issue.
"""
import csv, gzip, sys

args = sys.argv[1:]
if args and (args[0].endswith(".csv") or args[0].endswith(".gz")):
    fh = gzip.open(args[0], "rt") if args[0].endswith(".gz") else open(args[0])
    title = args[1] if len(args) > 1 else args[0]
else:
    fh, title = sys.stdin, (args[0] if args else "")
rows = list(csv.reader(fh))
hdr, units, vals = rows[0], rows[1], rows[2]
m = {h: (u, v) for h, u, v in zip(hdr, units, vals)}


def get(name):
    u, v = m.get(name, ("", ""))
    return f"{v} {u}".strip()


print(title)
print(f"  kernel: {get('Kernel Name') or get('launch__function_name')}  grid {get('launch__grid_size')} x block {get('launch__block_size')}, "
      f"{get('launch__registers_per_thread')}, cluster {get('launch__cluster_size') or '1'}")
for k in ("gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
          "lts__t_bytes.sum", "lts__t_bytes.sum.per_second", "lts__t_sectors.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "dram__bytes_read.sum.per_second", "sm__throughput.avg.pct_of_peak_sustained_elapsed"):
    if k in m:
        print(f"  {k:62s} {get(k)}")
try:
    dur_ms = float(m["gpu__time_duration.sum"][1]) * {"ms": 1.0, "us": 1e-3, "s": 1e3, "ns": 1e-6}.get(m["gpu__time_duration.sum"][0], 1.0)
    sect = float(m["lts__t_sectors.sum"][1])
    print(f"  {'L2 traffic (lts__t_sectors x 32 B)':62s} {sect * 32 / 1e6:.1f} MB per launch = {sect * 32 / (dur_ms * 1e-3) / 1e9:.1f} GB/s")
except (KeyError, ValueError):
    pass
print("  execution pipes, % of peak while active (IMAD / IMAD.WIDE issue on the fma pipe):")
for h in sorted(m):
    if h.startswith("sm__inst_executed_pipe_") and h.endswith(".avg.pct_of_peak_sustained_active"):
        v = float(m[h][1] or 0)
        if v >= 0.05:
            print(f"    {h[len('sm__inst_executed_pipe_'):-len('.avg.pct_of_peak_sustained_active')]:28s} {v:6.2f}")
print("  warp stalls per issued instruction:")
st = [(h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(m[h][1] or 0)) for h in m
      if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
for name, v in sorted(st, key=lambda kv: -kv[1])[:8]:
    print(f"    {name:28s} {v:6.3f}")
