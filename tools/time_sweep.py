"""Times one full sweep on the GPU (diagnostic)."""
import json, os, sys, time, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_05465_b200 as ssg
from paper_2405_05465_b200 import catalog
ssg.init(0)
d = tempfile.mkdtemp()
kw = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {}
path = catalog.write_search_config(d, **kw)
t0 = time.time(); s = ssg.SearchSession(path); t1 = time.time()
print("setup %.2fs configs %d" % (t1 - t0, s.num_configs), flush=True)
for rep in range(int(os.environ.get("REPS", "2"))):
    ssg.stats_reset(); t0 = time.time(); recs = s.run(); t1 = time.time()
    st = ssg.stats()
    print("sweep %.3fs  %.1f configs/s  stats %s" % (t1 - t0, s.num_configs / (t1 - t0), json.dumps(st)), flush=True)
out = ssg.search_finalize(path, recs)
print(out["summary"])
