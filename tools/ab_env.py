"""A/B of sweep environment knobs in one process (diagnostic): every setting must
give byte-identical records; prints sweep time per setting.
Usage: python tools/ab_env.py "SSG_SPEC_DEPTH=3,SSG_SPEC_LADDER=4 SSG_SPEC_DEPTH=2" [reps]"""
import hashlib, os, sys, time, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_05465_b200 as ssg
from paper_2405_05465_b200 import catalog

ssg.init(0)
path = catalog.write_search_config(tempfile.mkdtemp())
s = ssg.SearchSession(path)
settings = sys.argv[1].split()
# AB_SHARD="r/N": time one rank's shard of an N-GPU run (records hash per shard)
shard, nsh = (int(x) for x in os.environ.get("AB_SHARD", "0/1").split("/"))
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ref = None
s.run(shard, nsh)
for st in settings:
    env = dict(kv.split("=") for kv in st.split(","))
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    ts = []
    for r in range(reps):
        ssg.stats_reset(); t0 = time.perf_counter(); recs = s.run(shard, nsh); ts.append(time.perf_counter() - t0)
        h = hashlib.sha256(recs).hexdigest()[:16]
        ref = ref or h
        assert h == ref, ("records differ", st, h, ref)
    x = ssg.stats()
    print("%-40s sweep %s s | last sweep: launches %d units %d iters %.1fM | spec SLO %d used %d" % (
          st, " ".join("%.3f" % t for t in ts), x["launches_simulate"], x["units"],
          x["iterations"] / 1e6, x.get("spec_slo_runs", 0), x.get("spec_slo_used", 0)),
          flush=True)
    for k, v in old.items():
        if v is None: os.environ.pop(k, None)
        else: os.environ[k] = v
print("records identical across settings:", ref)
