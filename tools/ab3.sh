#!/bin/bash
cd "$(dirname "$0")/.."
for rep in 1 2; do
for lib in build/variants/v0_old.so build/variants/vb_allinline_noff.so build/variants/vc_allinline_ff.so; do
  echo "== $lib"
  SSG_LIB=$PWD/$lib REPS=2 timeout 300 python tools/time_sweep.py 2>&1 | grep -E "^sweep" | cut -c1-40
done
done
