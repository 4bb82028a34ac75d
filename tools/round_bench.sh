#!/bin/bash
# One GPU call: the bench line, the ncu launch list of a short bench run, one
# ncu --set full capture of sweep launch 2 and the k_predict metrics (diagnostic;
# outputs under gpurun_out/, summaries copied to profiles/ by hand).
cd "$(dirname "$0")/.."
TAG=${1:-r2}
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/launches_run_$TAG.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_bytes.sum.per_second,lts__t_sectors.avg.pct_of_peak_sustained_elapsed,l1tex__t_bytes.sum,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum \
  --clock-control none -k regex:"k_predict|k_bucket" --csv --log-file gpurun_out/kpredict_$TAG.csv python tools/pred_only.py > /dev/null 2>&1
tools/ncu_sweep_launch.sh 2 ${TAG}l2
