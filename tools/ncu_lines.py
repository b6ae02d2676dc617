#!/usr/bin/env python3
"""Aggregate ncu warp-stall samples per CUDA source line.

    ncu -i X.ncu-rep --page source --csv --print-source=cuda,sass > mix.csv
    python tools/ncu_lines.py mix.csv [top]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
samples = defaultdict(float)
execd = defaultdict(float)
text = {}
cur_file, cur_line = "?", None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 6:
        continue
    if r[0] not in ("", "-"):
        cur_line = (cur_file, int(r[0]))
        text[cur_line] = r[1][:90]
        continue
    if r[2].startswith("0x") and cur_line:
        samples[cur_line] += float(r[4] or 0)
        execd[cur_line] += float(r[7] or 0)
tot = sum(samples.values()) or 1
for key, s in sorted(samples.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100*s/tot:5.1f}%  {key[0]}:{key[1]:<5d} {text.get(key,'')}")


def reasons(path, top=15):
    """Stall-reason totals over the whole kernel (columns stall_*)."""
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    idx = {h: i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h}
    tot = defaultdict(float)
    for r in rows:
        if len(r) > 10 and r[2].startswith("0x"):
            for h, i in idx.items():
                tot[h] += float(r[i] or 0)
    s = sum(tot.values()) or 1
    for h, v in sorted(tot.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{100*v/s:5.1f}%  {h}")


if len(sys.argv) > 3 and sys.argv[3] == "reasons":
    reasons(sys.argv[1])


def active_lines(path, top=30):
    """Per source line: samples that are NOT barrier/cluster-barrier waits -- the critical path."""
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    ib = hdr.index("stall_barrier")
    samples = defaultdict(float)
    text = {}
    cur = None
    fname = "?"
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No" or len(r) < 10:
            continue
        if r[0] not in ("", "-"):
            cur = (fname, int(r[0]))
            text[cur] = r[1][:80]
            continue
        if r[2].startswith("0x") and cur:
            sass = r[3]
            if "CGABAR" in sass or "BAR.SYNC" in sass:
                continue
            samples[cur] += float(r[4] or 0) - float(r[ib] or 0)
    s = sum(samples.values()) or 1
    for key, v in sorted(samples.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{100*v/s:5.1f}%  {key[0]}:{key[1]:<5d} {text.get(key,'')}")


if len(sys.argv) > 3 and sys.argv[3] == "active":
    active_lines(sys.argv[1], int(sys.argv[2]))
