#!/bin/bash
# One `ncu --set full` capture (second launch) of the kernel each BASELINE workload selects. Run on the GPU box AFTER
# the same command exited 0 without ncu. The reports are summarised on the box (raw page -> tools/ncu_summary.py,
# source page -> tools/ncu_lines.py) and deleted: only the text summaries travel back (gpurun_out/ is capped at 64 MiB).
#   bash tools/ncu_all.sh [outdir]
set -u
out=${1:-gpurun_out/ncu_r02}
mkdir -p $out
cap() { # name regex title K N steps n_traj cluster
  python tools/one_launch.py $4 $5 $6 $7 auto $8 > $out/one_$1.log 2>&1 || { echo "$1: plain run failed"; return; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 --launch-skip 1 --launch-count 1 \
    -o /tmp/ncu_$1 -f python tools/one_launch.py $4 $5 $6 $7 auto $8 > $out/ncu_$1.log 2>&1
  echo "$1 ncu rc=$?"
  ncu -i /tmp/ncu_$1.ncu-rep --page raw --csv > /tmp/ncu_$1_raw.csv 2>/dev/null
  ncu -i /tmp/ncu_$1.ncu-rep --page source --csv --print-source=cuda,sass > /tmp/ncu_$1_src.csv 2>/dev/null
  python tools/ncu_summary.py /tmp/ncu_$1_raw.csv "$3" > $out/r02_ncu_$1_summary.txt 2>&1
  echo "--- stall samples per source line" >> $out/r02_ncu_$1_summary.txt
  python tools/ncu_lines.py /tmp/ncu_$1_src.csv 30 >> $out/r02_ncu_$1_summary.txt 2>&1
  gzip -c /tmp/ncu_$1_raw.csv > $out/r02_ncu_$1_raw.csv.gz
  rm -f /tmp/ncu_$1.ncu-rep /tmp/ncu_$1_src.csv
}
cap k500_mx mx "mx kernel, configs[1] K=500 N=200, one trajectory on a 16-CTA cluster, 100 steps" 500 200 100 1 16
cap ens100_warp warp "warp kernel, configs[4] (100,60), 4096 members, 10 steps" 100 60 10 4096 1
cap ens400_block block "block kernel, configs[4] (400,240), 4096 members, 2 steps" 400 240 2 4096 1
cap ens800_team team "team kernel, configs[4] (800,480), 4096 members, 1 step" 800 480 1 4096 1
cap k2200_grid grid "grid kernel, configs[2] K=2200 N=1000, one trajectory on 148 SMs, 2 steps" 2200 1000 2 1 16
