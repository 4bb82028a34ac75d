#!/bin/bash
# A/B of library build variants and env settings on the full cfg #4 sweep (diagnostic).
# usage: tools/ab_libs.sh "label=lib:ENV=VAL,ENV=VAL ..."
cd "$(dirname "$0")/.."
for spec in $1; do
  label=${spec%%=*}; rest=${spec#*=}; lib=${rest%%:*}; envs=${rest#*:}
  [ "$envs" = "$rest" ] && envs=""
  [ "$lib" = "default" ] && lib=paper_2405_05465_b200/libssg.so
  echo "== $label ($lib) $envs"
  env $(echo $envs | tr ',' ' ') SSG_LIB=$PWD/$lib REPS=3 timeout 300 python tools/time_sweep.py 2>&1 | grep -E "^sweep" | cut -c1-42
done
