#!/bin/bash
# One `ncu --set full` capture (second launch) of the kernel each BASELINE workload selects, plus the launch list
# of the default bench. Run on the GPU box AFTER the same commands exited 0 without ncu; reports land in gpurun_out/.
#   bash tools/ncu_all.sh
set -u
out=gpurun_out
cap() { # name regex K N steps n_traj cluster
  python tools/one_launch.py $3 $4 $5 $6 auto $7 > $out/one_$1.log 2>&1 || { echo "$1: plain run failed"; return; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 --launch-skip 1 --launch-count 1 \
    -o $out/r02_$1 -f python tools/one_launch.py $3 $4 $5 $6 auto $7 > $out/ncu_$1.log 2>&1
  echo "$1 rc=$?"
}
cap k500_mx mx 500 200 100 1 16
cap ens100_warp warp 100 60 10 4096 1
cap ens400_block block 400 240 2 4096 1
cap ens800_team team 800 480 1 4096 1
cap k2200_grid grid 2200 1000 2 1 16
