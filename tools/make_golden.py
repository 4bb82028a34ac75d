"""Generates tests/golden/ fixtures from the compiled REFERENCE (oracle/_ref).

Run in the build container (needs /root/reference compiled by `make -C oracle`):
    python tools/make_golden.py
For each case the reference trains the estimator (its own train()), predicts
the query set, and records the outputs under BOTH glibc libm contraction
variants -- the default (FMA on this host) in-process and the plain SSE2
variant in a child process with GLIBC_TUNABLES=glibc.cpu.hwcaps=-AVX2,-FMA.
Also records predict_batch goldens and a short simulation's batch log.
"""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2405_05465_b200 import catalog, OPS  # noqa: E402

SMALL = {"schema_version": 1, "name": "small", "num_layers": 4, "hidden_dim": 256,
         "num_q_heads": 8, "num_kv_heads": 8, "head_dim": 32, "mlp_dim": 1024,
         "vocab_size": 1000, "max_context": 4096, "param_bytes_per_element": 2,
         "attention_variant": "mha"}
TEST_GPU = {"schema_version": 1, "sku_name": "TEST-GPU", "peak_flops": 100e12,
            "mem_bandwidth": 1e12, "link_bandwidth": 2e11, "kernel_overhead": 2e-6,
            "device_mem": 16e9}
CASES = [  # (name, spec, device, tps, regressor, seed) -- test_estimator.cpp:11-43 fixtures
    ("small_interp", SMALL, TEST_GPU, [1, 2], "interp", 42),
    ("small_forest", SMALL, TEST_GPU, [1], "forest", 42),
    ("llama70b_h100_forest_tp4", catalog.MODELS["llama2_70b"], catalog.DEVICES["h100_80g"], [4], "forest", 3),
]


def queries(spec, tps, n=512, seed=0):
    rng = np.random.default_rng(seed)
    rows = []
    for tp in tps:
        kvb = 2 * (spec["num_kv_heads"] // tp) * spec["head_dim"] * spec["param_bytes_per_element"]
        for op in OPS:
            if op in ("allreduce", "allgather") and tp == 1:
                continue
            u = rng.random(n)
            f0 = np.floor(spec["max_context"] ** u)
            f1 = np.zeros(n)
            if op in ("attn_prefill", "attn_decode"):
                f1 = np.floor((512.0 * spec["max_context"]) ** rng.random(n)) * kvb
            elif op in ("allreduce", "allgather", "send_recv"):
                f0 = np.floor(1024.0 * 1048576.0 ** u)
            for a, b in zip(f0, f1):
                rows.append((OPS.index(op), tp, a, b))
    arr = np.array(rows)
    return arr[:, 0].astype(np.int32), arr[:, 1].astype(np.int64), arr[:, 2], arr[:, 3]


def evaluate(case_idx):
    name, spec, dev, tps, reg, seed = CASES[case_idx]
    est = ref.train(spec, dev, tps, reg, seed)
    e = ref.Estimator(est)
    ops, tp, f0, f1 = queries(spec, tps)
    out, bad, msg = e.predict(ops, tp, f0, f1)
    assert bad == -1, msg
    return est, (ops, tp, f0, f1), out


def child():
    idx = int(sys.argv[2])
    _, _, out = evaluate(idx)
    sys.stdout.write(json.dumps([v.hex() for v in out]))


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        return child()
    golden = {}
    for i, (name, spec, dev, tps, reg, seed) in enumerate(CASES):
        est, (ops, tp, f0, f1), out_default = evaluate(i)
        env = dict(os.environ, GLIBC_TUNABLES="glibc.cpu.hwcaps=-AVX2,-FMA")
        res = subprocess.run([sys.executable, __file__, "--child", str(i)], env=env, check=True,
                             capture_output=True, text=True)
        out_plain = np.array([float.fromhex(h) for h in json.loads(res.stdout)])
        golden[name + "__ops"] = ops
        golden[name + "__tp"] = tp
        golden[name + "__f0"] = f0
        golden[name + "__f1"] = f1
        golden[name + "__out_fma"] = out_default  # this container's libm is the FMA variant
        golden[name + "__out_plain"] = out_plain
        golden[name + "__est_sha"] = np.frombuffer(
            __import__("hashlib").sha256(est.encode()).digest(), dtype=np.uint8)
        diff = int(np.sum(out_default.view(np.uint64) != out_plain.view(np.uint64)))
        print("%-28s %6d queries, variants differ on %d" % (name, len(out_default), diff))
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "predict_golden.npz"), **golden)
    meta = {"cases": [{"name": c[0], "spec": c[1], "device": c[2], "tps": c[3], "regressor": c[4],
                       "seed": c[5]} for c in CASES],
            "generator": "tools/make_golden.py (reference compiled by oracle/Makefile)"}
    with open(os.path.join(ROOT, "tests", "golden", "predict_golden.json"), "w") as f:
        json.dump(meta, f, indent=1)


if __name__ == "__main__":
    main()
