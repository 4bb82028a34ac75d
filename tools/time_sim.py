"""Times one cfg #2 (or cfg #1) simulation through ssg.simulate (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2405_05465_b200 as ssg
from paper_2405_05465_b200 import catalog
ssg.init(0)
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if cfg == "cfg2":
    est = ssg.Estimator.train(catalog.MODELS["llama2_70b"], catalog.DEVICES["h100_80g"], [4], "interp", seed=0)
    pre, dec = ssg.synth_trace(catalog.zipf_histogram(), 10000, 42)
    cl = catalog.cluster_doc("llama2_70b", "h100_80g", tp=4, policy="sarathi_serve", max_batch_size=128, chunk_size=512)
    arr = ssg.poisson_arrivals(10000, 10.0, 0)
else:
    est = ssg.Estimator.train(catalog.MODELS["llama2_7b"], catalog.DEVICES["a100_80g"], [1], "interp", seed=0)
    L = catalog.fixture_chat_1k(); pre, dec = L[:, 0].astype(np.int64), L[:, 1].astype(np.int64)
    cl = catalog.cluster_doc("llama2_7b", "a100_80g", policy="vllm", max_batch_size=128)
    arr = ssg.poisson_arrivals(len(pre), 10.0, 5)
ids = np.arange(len(pre), dtype=np.int64)
for rep in range(3):
    ssg.stats_reset(); t0 = time.perf_counter()
    r = ssg.simulate(cl, est, ids, arr, pre, dec)
    t1 = time.perf_counter(); st = ssg.stats()
    print("rep %d wall %.3f s kernel %.3f s iterations %d" % (rep, t1 - t0, st["simulate_ms"] / 1e3, st["iterations"]), flush=True)
