"""Runs the exhaustive device-libm check (ssg_math_check) over the predictor's
whole integer feature domain for the cfg #4/#5 models, in this process's libm
mode, and prints one JSON line.  Used by tests/test_numerics_gpu.py, which runs
it once in the default ifunc mode and once with GLIBC_TUNABLES selecting the
SSE2 (non-FMA) glibc variant.

Domain (estimator.hpp:300-341, 113-119): every log1p input is an integer
multiple of a per-feature quantum -- 1 token (num_tokens), the KV bytes per
token of one block (kv_read_bytes = context tokens x 2 x elem x kv_heads/tp x
head_dim), or the payload bytes per token of a collective (payload_bytes =
tokens x hidden x elem, or x vocab/tp x elem) -- and lies inside the trained
box plus the 10 % extrapolation margin.  exp is checked on a 2^25-point grid
over [-25, 10], which covers every log-runtime the estimators produce."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import paper_2405_05465_b200 as ssg  # noqa: E402
from paper_2405_05465_b200 import catalog  # noqa: E402

MODELS = ("llama2_7b", "llama2_70b", "internlm_20b", "qwen_72b")


def domains():
    """{(quantum, count)}: progressions k * quantum, k in [0, count)."""
    out = set()
    for name in MODELS:
        spec = catalog.MODELS[name]
        e = spec["param_bytes_per_element"]
        tps = [tp for tp in (1, 2, 4) if spec["num_kv_heads"] % tp == 0]
        for dev in ("a100_80g", "h100_80g"):
            est = ssg.Estimator.train(spec, catalog.DEVICES[dev], tps, "interp", seed=0)
            doc = json.loads(est.to_json())
            for key, m in doc["ops"].items():
                tp = m["tp_degree"]
                for f, feat in enumerate(m["schema"]):
                    lo, hi = m["bbox_lo"][f], m["bbox_hi"][f]
                    upper = hi + 0.1 * (hi - lo)
                    if feat == "num_tokens":
                        quanta = [1]
                    elif feat == "kv_read_bytes":
                        quanta = [2 * e * (spec["num_kv_heads"] // tp) * spec["head_dim"]]
                    else:  # payload_bytes: allreduce / send_recv (hidden), allgather (vocab / tp)
                        quanta = [spec["hidden_dim"] * e, (spec["vocab_size"] // tp) * e]
                    for q in quanta:
                        out.add((q, int(math.floor(upper / q)) + 1))
    # keep the longest progression per quantum (shorter ones are prefixes)
    best = {}
    for q, n in out:
        best[q] = max(best.get(q, 0), n)
    return sorted(best.items())


def main():
    ssg.init(0)
    res = {"variant": ssg.math_variant(), "log1p": [], "exp": None}
    total = 0
    for q, n in domains():
        bad, first = ssg.math_check("log1p", 0.0, float(q), n)
        res["log1p"].append({"quantum": q, "values": n, "mismatches": bad,
                             "first": None if bad == 0 else first})
        total += n
    res["log1p_values"] = total
    n = 1 << 25
    bad, first = ssg.math_check("exp", -25.0, 35.0 / n, n)
    res["exp"] = {"values": n, "mismatches": bad, "first": None if bad == 0 else first}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
