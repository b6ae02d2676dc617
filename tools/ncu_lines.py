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
