"""TEST INFRASTRUCTURE: pure-Python restatement of the reference predictor path.

A second, independent statement of the arithmetic the GPU kernels implement,
written from the reference sources (cited per function) with Python floats
(IEEE binary64, no contraction) and the C libm through `math`, so it is
bit-comparable to the compiled reference on the same host.  It is pinned
against oracle/_ref (the reference itself) and against the golden vectors in
tests/golden/ by tests/test_oracle.py.  Small inputs only.
"""
from __future__ import annotations

import bisect
import math

OPS = ["qkv_proj", "attn_out_proj", "mlp_up_proj", "mlp_down_proj", "act_fn", "add_norm",
       "attn_prefill", "attn_decode", "allreduce", "allgather", "send_recv"]
TOKEN_OPS = OPS[:6]
COMM_OPS = OPS[8:]


def _clamp(v, lo, hi):
    # std::clamp(v, lo, hi)
    return lo if v < lo else (hi if hi < v else v)


def forest_regress(reg: dict, x) -> float:
    """ForestRegressor::predict / predict_tree (regressor.hpp:103-108, 256-264)."""
    s = 0.0
    nf = reg["num_features"]
    for t in reg["trees"]:
        node = 0
        feat, thr, left, right = t["feature"], t["threshold"], t["left"], t["right"]
        while feat[node] >= 0:
            node = left[node] if x[feat[node]] <= thr[node] else right[node]
        w = t["leaf_weights"][-feat[node] - 1]
        v = w[0]
        for f in range(nf):
            v += w[f + 1] * x[f]
        s += _clamp(v, reg["y_lo"], reg["y_hi"])
    return s / float(len(reg["trees"]))


def interp_regress(reg: dict, x) -> float:
    """GridInterpolator::predict (regressor.hpp:308-341)."""
    axes, values = reg["axes"], reg["values"]
    nf = len(axes)
    lo, frac = [0] * nf, [0.0] * nf
    for f in range(nf):
        ax = axes[f]
        if len(ax) == 1:
            continue
        hi = min(max(bisect.bisect_right(ax, x[f]), 1), len(ax) - 1)
        lo[f] = hi - 1
        frac[f] = _clamp((x[f] - ax[lo[f]]) / (ax[hi] - ax[lo[f]]), 0.0, 1.0)
    acc = 0.0
    for mask in range(1 << nf):
        w, flat, stride = 1.0, 0, 1
        for f in range(nf - 1, -1, -1):
            high = (mask >> f) & 1
            if len(axes[f]) == 1:
                high = 0
            w *= frac[f] if high else 1.0 - frac[f]
            flat += (lo[f] + high) * stride
            stride *= len(axes[f])
        acc += w * values[flat]
    return acc


class EstimatorError(ValueError):
    pass


def _fmt(v: float) -> str:
    return "%f" % v  # std::to_string(double)


def predict(est: dict, op: str, tp: int, feats) -> float:
    """EstimatorModel::predict (estimator.hpp:105-123)."""
    key = "%s@tp%d" % (op, tp)
    if key not in est["ops"]:
        raise EstimatorError("estimator: no trained model for op %s (profile and train must "
                             "cover the config's operators)" % key)
    m = est["ops"][key]
    x = []
    for f, name in enumerate(m["schema"]):
        v = feats[f]
        lo, hi = m["bbox_lo"][f], m["bbox_hi"][f]
        margin = 0.10 * (hi - lo)
        if not (v >= lo - margin and v <= hi + margin):
            raise EstimatorError(
                "estimator: feature %s=%s for %s outside extrapolation margin [%s, %s]"
                % (name, _fmt(v), key, _fmt(lo - margin), _fmt(hi + margin)))
        x.append(math.log1p(v))
    reg = m["regressor"]
    r = forest_regress(reg, x) if reg["type"] == "forest" else interp_regress(reg, x)
    return math.exp(r)


# ------------------------------------------------------------------ batches
def derive_operators(spec: dict, tp: int, pp: int = 1):
    """derive_operators (model_spec.hpp:203-266) as plain dicts."""
    lps = spec["num_layers"] // pp
    hq = spec["num_q_heads"] * spec["head_dim"]
    hkv = spec["num_kv_heads"] * spec["head_dim"]
    e = spec["param_bytes_per_element"]
    h, mlp = spec["hidden_dim"], spec["mlp_dim"]
    ops = []
    for op, i, o in [("qkv_proj", h, (hq + 2 * hkv) // tp), ("attn_out_proj", hq // tp, h),
                     ("mlp_up_proj", h, mlp // tp), ("mlp_down_proj", mlp // tp, h),
                     ("act_fn", mlp // tp, mlp // tp), ("add_norm", h, h)]:
        ops.append(dict(op=op, cls="token", count=lps, tp=tp, in_dim=i, out_dim=o, e=e))
    for op in ("attn_prefill", "attn_decode"):
        ops.append(dict(op=op, cls="seq", count=lps, tp=tp, qh=spec["num_q_heads"] // tp,
                        kvh=spec["num_kv_heads"] // tp, hd=spec["head_dim"], e=e))
    if tp > 1:
        ops.append(dict(op="allreduce", cls="comm", count=2 * lps, tp=tp, pay=h * e, e=e))
        ops.append(dict(op="allgather", cls="comm", count=1, tp=tp,
                        pay=(spec["vocab_size"] // tp) * e, e=e))
    if pp > 1:
        ops.append(dict(op="send_recv", cls="comm", count=1, tp=tp, pay=h * e, e=e))
    return ops


def equivalent_prefill_length(lengths) -> int:
    """estimator.hpp:38-46: llround(sqrt(sum p^2))."""
    sq = 0.0
    for p in lengths:
        sq += float(p) * float(p)
    r = math.sqrt(sq)
    t = math.floor(r)
    return int(t + 1) if r - t >= 0.5 else int(t)


def predict_batch(est: dict, ops, prefill_lengths, prefill_prior, decode_ctx) -> float:
    """predict_batch (estimator.hpp:294-348)."""
    total = float(len(decode_ctx) + sum(prefill_lengths))
    secs = 0.0
    for d in ops:
        count = float(d["count"])
        if d["cls"] == "token":
            secs += count * predict(est, d["op"], d["tp"], [total])
        elif d["cls"] == "seq":
            kvb = 2.0 * float(d["e"]) * float(d["kvh"] * d["hd"])
            if d["op"] == "attn_prefill":
                if not prefill_lengths:
                    continue
                n_eq = float(equivalent_prefill_length(prefill_lengths))
                prior = 0.0
                for c in prefill_prior:
                    prior += float(c)
                secs += count * predict(est, d["op"], d["tp"], [n_eq, prior * kvb])
            else:
                if not decode_ctx:
                    continue
                ctx = 0.0
                for c in decode_ctx:
                    ctx += float(c)
                secs += count * predict(est, d["op"], d["tp"], [float(len(decode_ctx)), ctx * kvb])
        else:
            secs += count * predict(est, d["op"], d["tp"], [total * float(d["pay"])])
    return secs
