#!/bin/bash
# ncu --set full of one k_simulate launch of the cfg #4 sweep plus its source
# pages (diagnostic).  usage: tools/ncu_sweep_launch.sh <launch-index> <tag>
cd "$(dirname "$0")/.."
L=${1:-1}; T=${2:-cap}
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_simulate \
  --launch-skip $L --launch-count 1 -o gpurun_out/ksim_$T python tools/time_sweep.py > gpurun_out/ncu_$T.log 2>&1
ncu -i gpurun_out/ksim_$T.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/ksim_${T}_sass.csv.gz
ncu -i gpurun_out/ksim_$T.ncu-rep --page raw --csv > gpurun_out/ksim_${T}_raw.csv 2>/dev/null
