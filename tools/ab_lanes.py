"""A/B of the sweep's lane settings in one process (diagnostic): every setting
must give byte-identical records; prints sweep time per setting.
Usage: python tools/ab_lanes.py "1:0 4:0 8:0 8:1 16:0" [reps]"""
import hashlib, os, sys, time, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_05465_b200 as ssg
from paper_2405_05465_b200 import catalog

ssg.init(0)
path = catalog.write_search_config(tempfile.mkdtemp())
s = ssg.SearchSession(path)
settings = (sys.argv[1] if len(sys.argv) > 1 else "1:0 8:0").split()
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ref = None
s.run()  # warm
for st in settings:
    lanes, block = st.split(":")
    os.environ["SSG_LANES"], os.environ["SSG_LANE_BLOCK"] = lanes, block
    ts = []
    for r in range(reps):
        ssg.stats_reset(); t0 = time.perf_counter(); recs = s.run(); ts.append(time.perf_counter() - t0)
        h = hashlib.sha256(recs).hexdigest()[:16]
        ref = ref or h
        assert h == ref, ("records differ", st, h, ref)
    x = ssg.stats()
    print("lanes %s block %s: sweep %s s | k_sim sum %.0f ms busy %.0f ms launches %d iters %.1fM"
          % (lanes, block, " ".join("%.3f" % t for t in ts), x["simulate_ms"], x["simulate_busy_ms"],
             x["launches_simulate"], x["iterations"] / 1e6), flush=True)
print("records identical across settings:", ref)
