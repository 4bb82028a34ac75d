set -x
for lib in paper_2405_05465_b200/libssg.so build/ab/libssg_fs0.so; do
  SSG_LIB=$PWD/$lib STEPS=5 timeout 300 python tools/time_predict.py 2>&1 | grep -E '"value"|ms_per_step|identical' | head -4
done
for pol in vllm sarathi_serve orca_plus all; do
  if [ $pol = all ]; then arg='{}'; else arg="{\"schedulers\": [\"$pol\"]}"; fi
  rm -f gpurun_out/units_$pol.txt
  SSG_DUMP_UNITS=gpurun_out/units_$pol.txt REPS=2 timeout 300 python tools/time_sweep.py "$arg" 2>&1 | grep -E "^sweep" | cut -c1-60
done
SSG_UNIT_SORT=1 REPS=2 timeout 300 python tools/time_sweep.py 2>&1 | grep -E "^sweep" | cut -c1-60
gzip -f gpurun_out/units_*.txt
