#!/usr/bin/env python3
"""Opcode mix and per-line instruction / stall shares of one ncu capture.
    python tools/ncu_mix.py X.ncu-rep <units (e.g. trajectory-orders) per launch> [top]
"""
import csv, subprocess, sys
from collections import defaultdict

rep, units = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
ops = defaultdict(float); samples = defaultdict(float); execd = defaultdict(float); text = {}
stall = defaultdict(float)
cur_file, cur, hdr = "?", None, None
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8: continue
    if r[0] not in ("", "-"):
        cur = (cur_file, int(r[0])); text[cur] = r[1][:95]; continue
    if r[2].startswith("0x") and cur:
        toks = r[3].split()
        op = toks[1] if toks[0].startswith("@") else toks[0]
        base = ".".join(op.split(".")[:2]) if op.startswith(("IMAD", "LDS", "STS", "SHFL")) else op.split(".")[0]
        n = float(r[7] or 0)
        ops[base] += n; execd[cur] += n; samples[cur] += float(r[4] or 0)
        for k, name in enumerate(hdr):
            if name.startswith("stall_") and "Not Issued" not in name and k < len(r):
                try: stall[name] += float(r[k] or 0)
                except ValueError: pass
tot = sum(ops.values()); ts = sum(samples.values()) or 1
print(f"instructions per unit: {tot / units:.1f}")
for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:18]:
    print(f"  {100 * v / tot:5.1f}%  {v / units:8.1f}/unit  {k}")
print("stall samples:", ", ".join(f"{k[6:]} {100 * v / ts:.1f}%" for k, v in sorted(stall.items(), key=lambda kv: -kv[1])[:8]))
print("--- top lines (inst share, sample share)")
for k, v in sorted(execd.items(), key=lambda kv: -samples[kv[0]])[:top]:
    print(f"{100 * v / tot:5.1f}% {100 * samples[k] / ts:5.1f}%  {k[0]}:{k[1]:<4d} {text.get(k, '')}")
