"""Phase timing of the bench's e2e call vs the resident session (diagnostic).
Usage: python tools/time_e2e.py [reps]"""
import os, sys, time, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_05465_b200 as ssg
from paper_2405_05465_b200 import catalog

ssg.init(0)
path = catalog.write_search_config(tempfile.mkdtemp())
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for r in range(reps):
    t0 = time.perf_counter(); s = ssg.SearchSession(path); t1 = time.perf_counter()
    recs = s.run(); t2 = time.perf_counter(); s.close(); t3 = time.perf_counter()
    out = ssg.search_finalize(path, recs); t4 = time.perf_counter()
    ssg.stats_reset()
    recs2 = ssg.search_shard(path, 0, 1); t5 = time.perf_counter()
    st = ssg.stats()
    print("rep %d: open %.3f run %.3f close %.3f finalize %.3f | search_shard %.3f (k_simulate %.3f)"
          % (r, t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, st["simulate_ms"] / 1e3), flush=True)
    assert recs == recs2
