for lib in build/ab/libssg_prev.so paper_2405_05465_b200/libssg.so; do
  echo "== $lib"
  for args in '{}' '{"model": "llama2_7b", "workload": "bwb_like"}' '{"model": "qwen_72b", "workload": "bwb_like"}'; do
    echo -n "$args: "; SSG_LIB=$PWD/$lib REPS=2 timeout 300 python tools/time_sweep.py "$args" 2>&1 | grep -E "^sweep" | tail -1 | cut -c1-40
  done
done
