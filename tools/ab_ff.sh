#!/bin/bash
# A/B of the previous commit's library (build/old) against the working tree on
# single simulations (cfg #1, cfg #2) and sweep shards (diagnostic).
cd "$(dirname "$0")/.."
[ "$TESTS" = 1 ] && python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for lib in ${LIBS:-build/old/libssg.so paper_2405_05465_b200/libssg.so}; do
  echo "== $lib"
  for c in cfg1 cfg2; do SSG_LIB=$PWD/$lib timeout 300 python tools/time_sim.py $c 2>&1 | tail -1; done
  for sh in ${SHARDS:-0/8 0/4 0/2 0/1}; do
    SSG_LIB=$PWD/$lib AB_SHARD=$sh timeout 300 python tools/ab_env.py "SHARD=$sh" 2 2>&1 | head -1
  done
done
