"""Per-iteration cost of one long simulation unit (diagnostic).

Simulates a single-replica cluster over a 2000-request chat-like trace at a low
arrival rate -- the shape of the sweep's critical-path probes -- and reports
device ms per simulated batch (one warp, no co-resident work)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2405_05465_b200 as ssg
from paper_2405_05465_b200 import catalog

ssg.init(0)
spec = catalog.MODELS["llama2_70b"]
rows = []
for policy, tp, pp, qps in [("vllm", 4, 4, 0.3), ("sarathi_serve", 4, 4, 0.3), ("orca_plus", 4, 2, 1.0),
                            ("vllm", 4, 1, 2.0)]:
    est = ssg.Estimator.train(spec, catalog.DEVICES["a100_80g"], [tp], "interp", 0)
    cl = catalog.cluster_doc("llama2_70b", "a100_80g", tp=tp, pp=pp, policy=policy, max_batch_size=32)
    rng = np.random.default_rng(7)
    n = 2000
    pre = np.maximum(1, np.round(rng.lognormal(np.log(417), 1.086, n))).astype(np.int64)
    dec = np.maximum(1, np.round(rng.lognormal(np.log(139), 0.973, n))).astype(np.int64)
    tot = pre + dec
    over = tot > 4096
    dec[over] = np.maximum(1, 4096 - np.minimum(pre[over], 4095))
    pre[over] = np.minimum(pre[over], 4096 - dec[over])
    arr = np.cumsum(rng.exponential(1.0 / qps, n))
    ssg.stats_reset()
    t0 = time.time()
    r = ssg.simulate(cl, est, np.arange(n), arr, pre, dec)
    t1 = time.time()
    st = ssg.stats()
    it = st["iterations"]
    rows.append(dict(policy=policy, tp=tp, pp=pp, qps=qps, iterations=it, kernel_ms=st["simulate_ms"],
                     us_per_iter=1e3 * st["simulate_ms"] / max(1, it), wall_s=t1 - t0))
    print(json.dumps(rows[-1]), flush=True)
