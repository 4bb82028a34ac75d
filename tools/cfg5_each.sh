for m in llama2_7b llama2_70b internlm_20b qwen_72b; do for t in chat_like arxiv_like bwb_like; do
  echo -n "$m $t: "; REPS=2 timeout 300 python tools/time_sweep.py "{\"model\": \"$m\", \"workload\": \"$t\"}" 2>&1 | grep -E "^sweep" | tail -1 | cut -c1-40
done; done
