"""Strong-scaling emulation on one B200 (diagnostic): every rank's shard of an
N-GPU sweep is evaluated here one after another; the N-GPU step time is the
slowest shard (ranks run concurrently on their own GPUs).  Compares the
cost-based (LPT) shard split with i % N striding and checks that the merged
records equal the one-GPU outcome byte for byte.
Usage: python tools/time_shards.py [cfg4|cfg5] [N ...]"""
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_05465_b200 as ssg  # noqa: E402
from paper_2405_05465_b200 import catalog  # noqa: E402

ssg.init(0)
work = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
ns = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
if work == "cfg4":
    paths = [catalog.write_search_config(tempfile.mkdtemp())]
else:
    paths = [catalog.write_search_config(tempfile.mkdtemp(), model=m, workload=t)
             for m in ("llama2_7b", "llama2_70b", "internlm_20b", "qwen_72b")
             for t in ("chat_like", "arxiv_like", "bwb_like")]
sessions = [ssg.SearchSession(p) for p in paths]
size = ssg.record_size()
whole = [ssg.search_finalize(p, s.run(0, 1)) for p, s in zip(paths, sessions)]  # warm + reference


def run_shard(r, n):
    if len(sessions) == 1:
        return [sessions[0].run(r, n)]
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(len(sessions)) as ex:
        return list(ex.map(lambda s: s.run(r, n), sessions))


for split in ("lpt", "stride"):
    os.environ["SSG_SHARD_SPLIT"] = split
    for n in ns:
        times, parts = [], [[] for _ in paths]
        for r in range(n):
            t0 = time.perf_counter()
            recs = run_shard(r, n)
            times.append(time.perf_counter() - t0)
            for k, x in enumerate(recs):
                parts[k].append(x)
        same = all(ssg.search_finalize(p, b"".join(x)) == w for p, x, w in zip(paths, parts, whole))
        counts = [len(x) // size for x in parts[0]]
        print("%-6s N=%d  max shard %.3f s  shards %s  configs/shard(sweep 0) %s  identical %s"
              % (split, n, max(times), " ".join("%.3f" % t for t in times), counts, same), flush=True)
