#!/bin/bash
# Round-end sweep: one bench line per BASELINE.json workload (1 GPU), each under its own timeout.
# Usage (GPU box): bash tools/bench_all.sh [outdir]
out=${1:-gpurun_out/sweep}
mkdir -p "$out"
for w in k50 k2200 k4200 ens100 ens200 ens400 ens800; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --cpu-seconds 10 \
    > "$out/bench_$w.json" 2> "$out/bench_$w.err"
  echo "$w rc=$?" >> "$out/status.txt"
done
