"""Fast-forward stretch statistics (diagnostic; needs a library built with
VARIANT_FLAGS=-DSSG_FF_STATS, passed as SSG_LIB).  Runs cfg #1, cfg #2 and a
sweep shard (AB_SHARD=r/N, default 0/8) and prints, for each, the number of
fast-forward calls, the iterations they committed, the total iterations and
the histogram of stretch lengths (0, 1, 2-3, 4-7, 8-15, 16-31, 32+); then zero-length reasons: arrival pre-filter, a runner finishing, bbox, memory/cost, arrival in the chain; and BatchStarts not tried: > 32 runners, requests waiting."""
import ctypes as C, os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2405_05465_b200 as ssg
from paper_2405_05465_b200 import _ffi, catalog

ssg.init(0)
L = _ffi.lib()
buf = (C.c_ulonglong * 16)()


def report(label):
    L.ssg_debug_ff_stats(buf, 1)
    st = ssg.stats()
    v = list(buf)
    print("%-10s ff_calls %d ff_iters %d of %d iterations (%.0f%%) hist %s zero-reasons %s not-tried %s" % (
        label, v[0], v[1], st["iterations"], 100.0 * v[1] / max(1, st["iterations"]), v[2:9], v[9:14], v[14:16]), flush=True)


L.ssg_debug_ff_stats(buf, 1)
for cfg in ("cfg1", "cfg2"):
    if cfg == "cfg2":
        est = ssg.Estimator.train(catalog.MODELS["llama2_70b"], catalog.DEVICES["h100_80g"], [4], "interp", seed=0)
        pre, dec = ssg.synth_trace(catalog.zipf_histogram(), 10000, 42)
        cl = catalog.cluster_doc("llama2_70b", "h100_80g", tp=4, policy="sarathi_serve", max_batch_size=128, chunk_size=512)
        arr = ssg.poisson_arrivals(10000, 10.0, 0)
    else:
        est = ssg.Estimator.train(catalog.MODELS["llama2_7b"], catalog.DEVICES["a100_80g"], [1], "interp", seed=0)
        F = catalog.fixture_chat_1k(); pre, dec = F[:, 0].astype(np.int64), F[:, 1].astype(np.int64)
        cl = catalog.cluster_doc("llama2_7b", "a100_80g", policy="vllm", max_batch_size=128)
        arr = ssg.poisson_arrivals(len(pre), 10.0, 5)
    ssg.stats_reset()
    ssg.simulate(cl, est, np.arange(len(pre), dtype=np.int64), arr, pre, dec)
    report(cfg)
shard, nsh = (int(x) for x in os.environ.get("AB_SHARD", "0/8").split("/"))
s = ssg.SearchSession(catalog.write_search_config(tempfile.mkdtemp()))
ssg.stats_reset()
s.run(shard, nsh)
report("shard %d/%d" % (shard, nsh))
