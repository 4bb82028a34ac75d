#!/bin/bash
# ncu times of k_select and k_probe_setup over one cfg #4 sweep under two library builds (diagnostic)
cd /root/repo
for lib in build/ab/libssg_pre_small.so paper_2405_05465_b200/libssg.so; do
  SSG_LIB=$PWD/$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_select|k_probe_setup" --csv --log-file gpurun_out/small_$(basename $lib .so).csv python tools/time_sweep.py > /dev/null 2>&1
done
