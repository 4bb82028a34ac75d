#!/bin/bash
cd "$(dirname "$0")/.."
for rep in 1 2; do
for lib in build/variants/v0_old.so paper_2405_05465_b200/libssg.so build/variants/v2_inline.so; do
  echo "== $lib"
  SSG_LIB=$PWD/$lib REPS=2 timeout 300 python tools/time_sweep.py 2>&1 | grep -E "^sweep" | cut -c1-40
done
done
SSG_LIB=$PWD/paper_2405_05465_b200/libssg.so SSG_NO_FASTFWD=1 REPS=2 timeout 300 python tools/time_sweep.py 2>&1 | grep -E "^sweep" | cut -c1-40
