#!/bin/bash
# A/B of library build variants on the GPU box (diagnostic).
cd "$(dirname "$0")/.."
for lib in paper_2405_05465_b200/libssg.so build/variants/v2_inline.so build/variants/v3_ffinline.so; do
  echo "== $lib"
  SSG_LIB=$PWD/$lib timeout 300 python tools/time_unit.py 2>&1 | python3 -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l); print('  unit %-14s pp%d us/iter %.2f' % (d['policy'], d['pp'], d['us_per_iter']))
    except Exception: print('  ', l.strip()[:200])
"
  SSG_LIB=$PWD/$lib REPS=2 timeout 300 python tools/time_sweep.py 2>&1 | grep -E "^sweep" | cut -c1-40
done
