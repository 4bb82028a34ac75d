for kw in '{}' '{"schedulers":["vllm"]}' '{"schedulers":["orca_plus"]}' '{"schedulers":["sarathi_serve"]}'; do
  echo "== $kw"
  REPS=2 SSG_TRACE_LANES=1 python tools/time_sweep.py "$kw" 2>&1 | grep -v "^  skipped\|^configs evaluated\|^optimum\|^no config" | tail -40
done
