"""Host-buffer predictor timing (diagnostic): pinned vs pageable, and raw copies."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2405_05465_b200 as ssg
from paper_2405_05465_b200 import catalog
ssg.init(0)
est = ssg.Estimator.train(catalog.MODELS["llama2_70b"], catalog.DEVICES["h100_80g"], [4], "forest", seed=3)
nq = 10_000_000
rng = np.random.default_rng(0)
ops = ("attn_prefill", "attn_decode", "mlp_up_proj")
which = rng.integers(0, 3, nq)
slots = np.array([est.slot(o, 4) for o in ops], dtype=np.int32)[which]
f0 = np.floor(4096.0 ** rng.random(nq)); f1 = np.floor((512.0 * 4096.0) ** rng.random(nq)) * 1024.0
f1[which == 2] = 0.0
pin = [torch.from_numpy(a).pin_memory() for a in (slots, f0, f1)]
out = torch.empty(nq, dtype=torch.float64).pin_memory()
for label, args in (("pinned", [t.numpy() for t in pin] + [out.numpy()]), ("pageable", [slots, f0, f1, np.empty(nq)])):
    ts = []
    for _ in range(4):
        t0 = time.perf_counter(); est.predict_mixed(args[0], args[1], args[2], out=args[3]); ts.append(time.perf_counter() - t0)
    print(label, " ".join("%.2f" % (1e3 * t) for t in ts), "ms")
d = torch.empty(nq * 3, dtype=torch.float64, device="cuda")
h = torch.empty(nq * 3, dtype=torch.float64).pin_memory()
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d[: nq * 2 + nq // 2].copy_(h[: nq * 2 + nq // 2], non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    h[:nq].copy_(d[:nq], non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    print("raw H2D 200MB %.2f ms, D2H 80MB %.2f ms" % (1e3 * (t1 - t0), 1e3 * (t2 - t1)))
