"""K1/K2 parity: GPU EstimatorModel::predict vs the compiled reference, bit for bit.

Reference: estimator.hpp:105-123, regressor.hpp:103-108,256-264,308-341.
The oracle is the reference library itself (oracle/_ref), trained with the
reference's own train(); the GPU path loads that same JSON.
"""
import numpy as np
import pytest

from paper_2405_05465_b200 import catalog, OPS

pytestmark = pytest.mark.gpu


def queries(op, kvb, n, rng):
    """Feature draws shaped like the BASELINE cfg #3 microbench plus grid/edge points."""
    u = rng.random(n)
    f0 = np.floor(4096.0 ** u)
    f1 = None
    if op in ("attn_prefill", "attn_decode"):
        f1 = np.floor((512.0 * 4096.0) ** rng.random(n)) * kvb
        f1[:5] = [0.0, kvb, 512 * 4096 * kvb, 2 * kvb, 1.0]
    elif op in ("allreduce", "allgather", "send_recv"):
        f0 = np.floor(1024.0 * 1048576.0 ** u)
        f0[:3] = [1024.0, 2.0 ** 30, 3.0 * 2 ** 20]
    f0[:2] = [1.0, 4096.0] if op not in ("allreduce", "allgather", "send_recv") else f0[:2]
    return f0, f1


@pytest.mark.parametrize("model,dev,tps,reg", [
    ("llama2_70b", "h100_80g", [1, 2, 4], "interp"),
    ("llama2_70b", "h100_80g", [4], "forest"),
    ("llama2_7b", "a100_80g", [1, 2], "forest"),
    ("internlm_20b", "a100_80g", [1, 2, 4], "interp"),
])
def test_predict_bit_exact(ssg, ref, model, dev, tps, reg):
    est_json = ref.train(catalog.MODELS[model], catalog.DEVICES[dev], tps, reg, 11)
    mine = ssg.Estimator.from_json(est_json)
    theirs = ref.Estimator(est_json)
    rng = np.random.default_rng(5)
    spec = catalog.MODELS[model]
    for tp in tps:
        kvb = 2 * (spec["num_kv_heads"] // tp) * spec["head_dim"] * spec["param_bytes_per_element"]
        for op in OPS:
            if mine.slot(op, tp) < 0:
                continue
            f0, f1 = queries(op, kvb, 4000, rng)
            got = mine.predict(op, tp, f0, f1)
            want, bad, msg = theirs.predict(OPS.index(op), tp, f0, f1)
            assert bad == -1, msg
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (op, tp)


def test_predict_mixed_and_errors(ssg, ref):
    spec, dev = catalog.MODELS["llama2_70b"], catalog.DEVICES["h100_80g"]
    est_json = ref.train(spec, dev, [4], "forest", 3)
    mine = ssg.Estimator.from_json(est_json)
    theirs = ref.Estimator(est_json)
    rng = np.random.default_rng(9)
    kvb = 2 * 2 * 128 * 2
    n = 30000
    ops = rng.choice([OPS.index("attn_prefill"), OPS.index("attn_decode"), OPS.index("mlp_up_proj")], n)
    f0 = np.floor(4096.0 ** rng.random(n))
    f1 = np.floor((512.0 * 4096.0) ** rng.random(n)) * kvb
    slots = np.array([mine.slot(OPS[o], 4) for o in ops], dtype=np.int32)
    got = mine.predict_mixed(slots, f0, f1)
    want, bad, msg = theirs.predict(ops, 4, f0, f1)
    assert bad == -1
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))

    # guard violations: the lowest failing index wins, message verbatim
    f0b = f0.copy()
    f0b[[17, 400]] = [5000.0, 1e9]
    with pytest.raises(ssg.InputError) as ei:
        mine.predict_mixed(slots, f0b, f1)
    _, bad, msg = theirs.predict(ops, 4, f0b, f1)
    assert bad == 17
    assert str(ei.value) == msg
    f1b = f1.copy()
    i = int(np.nonzero(ops == OPS.index("attn_decode"))[0][3])
    f1b[i] = -1e12
    with pytest.raises(ssg.InputError) as ei:
        mine.predict_mixed(slots, f0, f1b)
    _, bad, msg = theirs.predict(ops, 4, f0, f1b)
    assert bad == i and str(ei.value) == msg


def test_untrained_op_message(ssg, ref):
    est_json = ref.train(catalog.MODELS["llama2_7b"], catalog.DEVICES["a100_80g"], [1], "interp", 0)
    mine = ssg.Estimator.from_json(est_json)
    with pytest.raises(ssg.InputError) as ei:
        mine.predict("allreduce", 2, np.array([4096.0]))
    assert str(ei.value) == ("estimator: no trained model for op allreduce@tp2 "
                             "(profile and train must cover the config's operators)")


def test_predict_mixed_chunked_pinned(ssg, ref):
    """Host-buffer predictions from pinned memory stream through 1M-query chunks on
    three streams: still bit-exact, and an error in a late chunk reports its global
    index with the reference's message; invalid slots and a missing f1 are caught
    in the kernel and raised before any prediction error."""
    import torch

    spec, dev = catalog.MODELS["llama2_70b"], catalog.DEVICES["h100_80g"]
    est_json = ref.train(spec, dev, [4], "interp", 3)
    mine = ssg.Estimator.from_json(est_json)
    theirs = ref.Estimator(est_json)
    rng = np.random.default_rng(4)
    n = 3 * (1 << 20) + 12345
    ops = rng.choice([OPS.index("attn_prefill"), OPS.index("attn_decode"), OPS.index("mlp_up_proj")], n)
    slots = np.array([mine.slot(OPS[o], 4) for o in range(len(OPS))], dtype=np.int32)[ops]
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    f0 = pin(np.floor(4096.0 ** rng.random(n)))
    f1 = pin(np.floor((512.0 * 4096.0) ** rng.random(n)) * 1024.0)
    slots_p = pin(slots)
    out = pin(np.zeros(n))
    got = mine.predict_mixed(slots_p, f0, f1, out=out)
    sample = rng.choice(n, 200000, replace=False)
    want, bad, _ = theirs.predict(ops[sample], 4, f0[sample], f1[sample])
    assert bad == -1
    assert np.array_equal(got[sample].view(np.uint64), want.view(np.uint64))
    # a guard violation in the third chunk
    i = 2 * (1 << 20) + 777
    f0[i] = 1e9
    with pytest.raises(ssg.InputError) as ei:
        mine.predict_mixed(slots_p, f0, f1, out=out)
    _, bad, msg = theirs.predict(ops[i:i + 1], 4, f0[i:i + 1], f1[i:i + 1])
    assert str(ei.value) == msg
    # an invalid slot wins over the guard violation, whatever its index
    slots_p[i + 5] = 999
    with pytest.raises(ssg.InputError, match="query %d has no trained model slot" % (i + 5)):
        mine.predict_mixed(slots_p, f0, f1, out=out)
    slots_p[i + 5] = slots[i + 5]
    with pytest.raises(ssg.InputError, match="two-feature models need f1"):
        mine.predict_mixed(slots_p, f0, None, out=out)


@pytest.mark.parametrize("model,dev,tps,seed", [
    ("llama2_7b", "a100_80g", [1], 42),          # the golden case small_forest
    ("llama2_70b", "h100_80g", [4], 3),          # cfg #3's estimator
    ("internlm_20b", "h100_80g", [1, 2], 21),
    ("qwen_72b", "a100_80g", [1, 2, 4], 7),
])
def test_device_forest_training_matches_reference(ssg, ref, model, dev, tps, seed):
    """(f)3: every forest -- hold-out probes and final models -- grows on the
    GPU (train.cu, one warp per tree) and the estimator JSON equals the
    reference's train() byte for byte (regressor.hpp:82-254, estimator.hpp:201-275)."""
    spec, device = catalog.MODELS[model], catalog.DEVICES[dev]
    want = ref.train(spec, device, tps, "forest", seed)
    got = ssg.Estimator.train(spec, device, tps, "forest", seed=seed).to_json()
    assert got == want


def test_device_forest_training_golden_sha():
    """The forest cases of tests/golden (reference estimator sha256) reproduced by the GPU trainer."""
    import hashlib
    import json
    import os

    import paper_2405_05465_b200 as ssg

    ssg.init(0)
    gdir = os.path.join(os.path.dirname(__file__), "golden")
    meta = json.load(open(os.path.join(gdir, "predict_golden.json")))
    data = np.load(os.path.join(gdir, "predict_golden.npz"))
    for case in meta["cases"]:
        if case["regressor"] != "forest":
            continue
        text = ssg.Estimator.train(case["spec"], case["device"], case["tps"], "forest",
                                   case["seed"]).to_json()
        assert hashlib.sha256(text.encode()).digest() == bytes(data[case["name"] + "__est_sha"])
