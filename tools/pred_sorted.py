"""Does grouping predictor queries by model help k_predict? (diagnostic)
Times 10M mixed queries as generated vs the same queries sorted by slot."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2405_05465_b200 as ssg
from paper_2405_05465_b200 import catalog
ssg.init(0)
dev = torch.device("cuda", 0)
est = ssg.Estimator.train(catalog.MODELS["llama2_70b"], catalog.DEVICES["h100_80g"], [4], "forest", seed=3)
nq = 10_000_000
rng = np.random.default_rng(0)
ops = ("attn_prefill", "attn_decode", "mlp_up_proj")
which = rng.integers(0, 3, nq)
slots = np.array([est.slot(o, 4) for o in ops], dtype=np.int32)[which]
f0 = np.floor(4096.0 ** rng.random(nq)); f1 = np.floor((512.0 * 4096.0) ** rng.random(nq)) * 1024.0
f1[which == 2] = 0.0
order_slot = np.argsort(slots, kind="stable")
order_full = np.lexsort((f1, f0, slots))
b0 = np.minimum(63, (np.log2(f0 + 1.0) * (64 / 12.0)).astype(np.int64))
b1 = np.minimum(63, (np.log2(f1 / 1024.0 + 1.0) * (64 / 21.0)).astype(np.int64))
order_b64 = np.argsort(slots.astype(np.int64) * 64 + b0, kind="stable")
order_b2 = np.argsort((slots.astype(np.int64) * 64 + b0) * 64 + b1, kind="stable")
order_b2c = np.argsort((slots.astype(np.int64) * 16 + b0 // 4) * 16 + b1 // 4, kind="stable")
for label, order in (("mixed", np.arange(nq)), ("by slot", order_slot), ("by slot, f0, f1", order_full),
                     ("slot x f0/64", order_b64), ("slot x f0/64 x f1/64", order_b2),
                     ("slot x f0/16 x f1/16", order_b2c)):
    d = [torch.from_numpy(np.ascontiguousarray(a[order])).to(dev) for a in (slots, f0, f1)]
    out = torch.empty(nq, dtype=torch.float64, device=dev)
    err = torch.full((1,), -1, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    ts = []
    for i in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); est.predict_device(nq, d[0].data_ptr(), 0, d[1].data_ptr(), d[2].data_ptr(), out.data_ptr(), err.data_ptr(), st); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print("%-16s %.3f ms  %.3f Gq/s" % (label, min(ts[1:]), nq / min(ts[1:]) / 1e6))
