"""K3 parity: GPU replica simulation vs the compiled reference run_simulation.

Checks, on identical inputs: every scheduled batch (replica, clock, KV units
allocated, entries with chunk/prior/context) -- the reference SimObserver
payload, sim.hpp:230 -- per-request records incl. every emission time,
replica aggregates, span, and the metrics report.  Bit-exact except total
model flops / MFU (summed across independent replicas in a different order;
north_star tolerance 1e-6 relative).
"""
import json

import numpy as np
import pytest

from paper_2405_05465_b200 import catalog

pytestmark = pytest.mark.gpu

_EST = {}


def estimators(ssg, ref, model, dev, tps, reg="interp", seed=3):
    key = (model, dev, tuple(tps), reg, seed)
    if key not in _EST:
        text = ref.train(catalog.MODELS[model], catalog.DEVICES[dev], tps, reg, seed)
        _EST[key] = (ssg.Estimator.from_json(text), ref.Estimator(text))
    return _EST[key]


def trace_fixture(n, qps, seed, scale_decode=1.0):
    lengths = catalog.fixture_chat_1k()
    idx = np.arange(n) % len(lengths)
    pre = lengths[idx, 0].astype(np.int64)
    dec = np.maximum(1, (lengths[idx, 1] * scale_decode).astype(np.int64))
    rng = np.random.default_rng(seed)
    arr = np.cumsum(rng.exponential(1.0 / qps, n))
    return np.arange(n, dtype=np.int64), arr, pre, dec


def by_replica(batches):
    out = {}
    for b in batches:
        out.setdefault(b["replica"], []).append(b)
    return out


def assert_same(mine, theirs, flops_rtol=1e-9):
    assert "probe_infeasible" not in mine and "probe_infeasible" not in theirs
    # batch logs, per replica in order
    bm, bt = by_replica(mine["batches"]), by_replica(theirs["batches"])
    assert sorted(bm) == sorted(bt)
    for r in bt:
        assert len(bm[r]) == len(bt[r]), ("batches", r)
        for k, (a, b) in enumerate(zip(bm[r], bt[r])):
            assert a["now"] == b["now"] and a["kv"] == b["kv"] and a["entries"] == b["entries"], (r, k, a, b)
    for a, b in zip(mine["requests"], theirs["requests"]):
        assert a == b, (a["id"], {k: (a[k], b[k]) for k in a if a[k] != b[k]})
    assert mine["replicas"] == theirs["replicas"]
    assert mine["simulated_span"] == theirs["simulated_span"]
    assert mine["total_model_flops"] == pytest.approx(theirs["total_model_flops"], rel=flops_rtol)
    rm, rt = mine["report"], theirs["report"]
    for k in ("scheduling_delay", "ttft", "tbt", "e2e", "normalized"):
        for q in ("p50", "p90", "p95", "p99"):
            assert rm[k][q] == rt[k][q], (k, q)
        assert rm[k]["mean"] == pytest.approx(rt[k]["mean"], rel=1e-12, abs=0)
    for k in ("kv_utilization_peak", "busy_fraction", "preemptions"):
        assert rm[k] == pytest.approx(rt[k], rel=1e-12), k
    assert rm["mfu"] == pytest.approx(rt["mfu"], rel=flops_rtol)
    assert mine["requests_csv"] == theirs["requests_csv"]


def run_both(ssg, mine_est, ref_est, cluster, trace, **kw):
    ids, arr, pre, dec = trace
    mine = ssg.simulate(cluster, mine_est, ids, arr, pre, dec, record_batches=True, **kw)
    theirs = ref_est.simulate(cluster, ids, arr, pre, dec, record_batches=True, **kw)
    return mine, theirs


@pytest.mark.parametrize("qps", [5.0, 10.0])
def test_cfg1_vllm_7b(ssg, ref, qps):
    """BASELINE cfg #1: LLaMA2-7B TP1, one replica, vLLM bs128, the 1K fixture."""
    m, t = estimators(ssg, ref, "llama2_7b", "a100_80g", [1])
    cluster = catalog.cluster_doc("llama2_7b", "a100_80g", policy="vllm", max_batch_size=128)
    mine, theirs = run_both(ssg, m, t, cluster, trace_fixture(1000, qps, 5))
    assert_same(mine, theirs)


def baseline_trace(ssg, lengths, qps, seed):
    """A trace built the reference's way: poisson_arrivals(qps, seed) over the lengths."""
    pre, dec = lengths
    n = len(pre)
    return (np.arange(n, dtype=np.int64), ssg.poisson_arrivals(n, qps, seed),
            np.asarray(pre, dtype=np.int64), np.asarray(dec, dtype=np.int64))


@pytest.mark.parametrize("qps", [5.0, 10.0])
def test_cfg1_fixture_poisson(ssg, ref, qps):
    """BASELINE cfg #1 exactly: the 1K chat fixture with poisson_arrivals(qps, seed 5)."""
    m, t = estimators(ssg, ref, "llama2_7b", "a100_80g", [1])
    cluster = catalog.cluster_doc("llama2_7b", "a100_80g", policy="vllm", max_batch_size=128)
    lengths = catalog.fixture_chat_1k()
    mine, theirs = run_both(ssg, m, t, cluster, baseline_trace(ssg, (lengths[:, 0], lengths[:, 1]), qps, 5))
    assert_same(mine, theirs)


@pytest.mark.slow
@pytest.mark.parametrize("qps", [10.0])
def test_cfg2_sarathi_70b_zipf_10k(ssg, ref, qps):
    """BASELINE cfg #2 at full size: LLaMA2-70B H100 TP4, Sarathi-Serve chunk 512,
    the 10K-request Zipf histogram trace (synth seed 42), poisson_arrivals seed 0.
    Every batch, every emission time and the report agree with the reference."""
    m, t = estimators(ssg, ref, "llama2_70b", "h100_80g", [4], seed=0)
    cluster = catalog.cluster_doc("llama2_70b", "h100_80g", tp=4, policy="sarathi_serve",
                                  max_batch_size=128, chunk_size=512)
    lengths = ssg.synth_trace(catalog.zipf_histogram(), 10000, 42)
    mine, theirs = run_both(ssg, m, t, cluster, baseline_trace(ssg, lengths, qps, 0))
    assert_same(mine, theirs)
    assert len(theirs["requests"]) == 10000


TIGHT = dict(catalog.DEVICES["a100_80g"], device_mem=30e9)


@pytest.mark.parametrize("policy,block_size", [("vllm", 24), ("sarathi_serve", 7), ("orca_plus", 1),
                                                ("vllm", 32)])
def test_block_sizes(ssg, ref, policy, block_size):
    """Block accounting for power-of-two and other block sizes (the device divides
    by a non-power-of-two block size with a 64-bit multiply-high), under memory
    pressure so shortfalls, watermarks and preemptions depend on the rounding."""
    m, t = estimators(ssg, ref, "llama2_7b", "a100_80g", [1])
    extra = {"chunk_size": 384} if policy == "sarathi_serve" else {}
    cluster = catalog.cluster_doc("llama2_7b", TIGHT, policy=policy, max_batch_size=64,
                                  block_size=block_size, **extra)
    mine, theirs = run_both(ssg, m, t, cluster, trace_fixture(500, 8.0, 3))
    assert_same(mine, theirs)


@pytest.mark.parametrize("policy,extra", [
    ("vllm", {}), ("orca_plus", {}), ("lightllm", {}),
    ("sarathi_serve", {"chunk_size": 512}), ("faster_transformer", {}),
])
def test_policies_under_memory_pressure(ssg, ref, policy, extra):
    """Acceptance #4 shape: a tight device forces watermark stalls and preemptions."""
    m, t = estimators(ssg, ref, "llama2_7b", "a100_80g", [1])
    cluster = catalog.cluster_doc("llama2_7b", TIGHT, policy=policy, max_batch_size=64, **extra)
    mine, theirs = run_both(ssg, m, t, cluster, trace_fixture(600, 8.0, 11))
    assert_same(mine, theirs)
    if policy == "vllm":
        assert theirs["report"]["preemptions"] > 0


@pytest.mark.parametrize("routing,replicas,n,qps", [("round_robin", 3, 900, 14.0),
                                                    ("least_outstanding", 3, 900, 14.0),
                                                    ("deferred", 4, 900, 14.0),
                                                    ("least_outstanding", 40, 3000, 400.0),
                                                    ("deferred", 40, 3000, 400.0)])
def test_routing(ssg, ref, routing, replicas, n, qps):
    """Routers, including more replicas than a warp has lanes (argmins run 32
    replicas per pass)."""
    m, t = estimators(ssg, ref, "llama2_7b", "a100_80g", [1])
    cluster = catalog.cluster_doc("llama2_7b", "a100_80g", replicas=replicas, routing=routing,
                                  policy="vllm", max_batch_size=32)
    mine, theirs = run_both(ssg, m, t, cluster, trace_fixture(n, qps, 2))
    assert_same(mine, theirs)


@pytest.mark.parametrize("tp,pp,policy", [(4, 1, "sarathi_serve"), (2, 2, "vllm"), (1, 4, "orca_plus"),
                                         (1, 5, "sarathi_serve"), (1, 16, "vllm"),
                                         (1, 20, "sarathi_serve"), (2, 40, "vllm"), (1, 80, "orca_plus")])
def test_70b_parallelism(ssg, ref, tp, pp, policy):
    """cfg #2 shape (70B, Sarathi cs512) plus pipeline microbatching; pp above 16
    takes the general latency path with its microbatch scratch in HBM."""
    m, t = estimators(ssg, ref, "llama2_70b", "h100_80g", [1, 2, 4])
    cluster = catalog.cluster_doc("llama2_70b", "h100_80g", tp=tp, pp=pp, policy=policy,
                                  max_batch_size=128, chunk_size=512, cpu_overhead=1e-4)
    mine, theirs = run_both(ssg, m, t, cluster, trace_fixture(700, 6.0, 4))
    assert_same(mine, theirs)


@pytest.mark.parametrize("max_batch", [3_000_000, 1 << 40])
def test_unbounded_max_batch(ssg, ref, max_batch):
    """A batch cap above any unit's request count (the reference accepts any
    int64 >= 1): queues are sized by min(max_batch_size, requests)."""
    m, t = estimators(ssg, ref, "llama2_7b", "a100_80g", [1])
    cluster = catalog.cluster_doc("llama2_7b", "a100_80g", policy="vllm", max_batch_size=max_batch)
    mine, theirs = run_both(ssg, m, t, cluster, trace_fixture(300, 20.0, 9))
    assert_same(mine, theirs)


def test_forest_regressor_sim(ssg, ref):
    m, t = estimators(ssg, ref, "llama2_7b", "a100_80g", [1], reg="forest")
    cluster = catalog.cluster_doc("llama2_7b", "a100_80g", policy="sarathi_serve", chunk_size=1024)
    mine, theirs = run_both(ssg, m, t, cluster, trace_fixture(400, 4.0, 8))
    assert_same(mine, theirs)


def test_probe_abort_matches(ssg, ref):
    """SimOptions abort (sim.hpp:231-240): same verdict as the reference."""
    m, t = estimators(ssg, ref, "llama2_7b", "a100_80g", [1])
    cluster = catalog.cluster_doc("llama2_7b", "a100_80g", replicas=2, policy="vllm")
    for qps, expect in [(60.0, True), (2.0, False)]:
        mine, theirs = run_both(ssg, m, t, cluster, trace_fixture(500, qps, 1),
                                abort_delay=5.0, abort_max_late=5)
        assert bool(mine.get("probe_infeasible")) == bool(theirs.get("probe_infeasible")) == expect


def test_enqueue_capacity_error(ssg, ref):
    m, t = estimators(ssg, ref, "llama2_7b", "a100_80g", [1])
    tiny = dict(catalog.DEVICES["a100_80g"], device_mem=15.2e9)
    cluster = catalog.cluster_doc("llama2_7b", tiny, policy="vllm")
    ids, arr, pre, dec = trace_fixture(50, 1.0, 0)
    pre[7] = 9000  # > the 369 blocks x 16 tokens this device leaves for KV
    with pytest.raises(ssg.InputError) as ei:
        ssg.simulate(cluster, m, ids, arr, pre, dec)
    from oracle.ref import RefError
    with pytest.raises(RefError) as er:
        t.simulate(cluster, ids, arr, pre, dec)
    assert str(ei.value) == str(er.value)


def test_predict_batch_parity(ssg, ref):
    m, t = estimators(ssg, ref, "llama2_70b", "h100_80g", [1, 2, 4])
    rng = np.random.default_rng(3)
    batches = []
    for _ in range(300):
        npf = int(rng.integers(0, 5))
        nd = int(rng.integers(0 if npf else 1, 200))
        pl = rng.integers(1, 1024, npf).tolist()
        pp = rng.integers(0, 3000, npf).tolist()
        dc = rng.integers(1, 4096, nd).tolist()
        batches.append((pl, pp, dc))
    batches.append(([3, 4], [0, 0], []))       # sqrt(3^2+4^2) = 5 (test_estimator.cpp:85-90)
    batches.append(([100] * 4, [0] * 4, []))   # -> 200
    spec = catalog.MODELS["llama2_70b"]
    for tp in (1, 2, 4):
        s_m, f_m = m.predict_batch(spec, tp, batches)
        s_t, f_t, res = t.predict_batch(spec, tp, batches)
        assert res == {}
        assert np.array_equal(s_m.view(np.uint64), s_t.view(np.uint64))
        assert np.array_equal(f_m.view(np.uint64), f_t.view(np.uint64))


def test_bbox_error_inside_a_batch(ssg, ref):
    """A decode batch whose KV volume leaves the trained box (estimator.hpp:115-119)
    surfaces the reference's exact Error from inside the simulation (token-table
    path: tokens stay in range, the attention feature does not)."""
    tiny = dict(catalog.MODELS["llama2_7b"], name="tiny-ctx", max_context=128)
    text = ref.train(tiny, catalog.DEVICES["a100_80g"], [1], "interp", 0)
    m, t = ssg.Estimator.from_json(text), ref.Estimator(text)
    cluster = catalog.cluster_doc(tiny, "a100_80g", policy="sarathi_serve", chunk_size=128,
                                  max_batch_size=128)
    n = 120
    ids = np.arange(n, dtype=np.int64)
    arr = np.arange(n, dtype=np.float64) * 1e-3
    pre = np.full(n, 300, dtype=np.int64)
    dec = np.full(n, 2000, dtype=np.int64)
    from oracle.ref import RefError
    with pytest.raises(RefError) as er:
        t.simulate(cluster, ids, arr, pre, dec)
    with pytest.raises(ssg.InputError) as ei:
        ssg.simulate(cluster, m, ids, arr, pre, dec)
    assert "attn_decode@tp1 outside extrapolation margin" in str(er.value)
    assert str(ei.value) == str(er.value)


def test_simulate_run_binary_outputs(ssg, ref):
    """ssg_simulate_run (binary outputs) agrees with the JSON path and the reference."""
    m, t = estimators(ssg, ref, "llama2_7b", "a100_80g", [1])
    cluster = catalog.cluster_doc("llama2_7b", "a100_80g", policy="sarathi_serve", max_batch_size=64,
                                  chunk_size=256)
    lengths = catalog.fixture_chat_1k()
    ids, arr, pre, dec = baseline_trace(ssg, (lengths[:, 0], lengths[:, 1]), 10.0, 5)
    run = ssg.simulate_run(cluster, m, ids, arr, pre, dec)
    theirs = t.simulate(cluster, ids, arr, pre, dec)
    for i, q in enumerate(theirs["requests"]):
        assert run.first_scheduled[i] == q["first_scheduled"] and run.first_token[i] == q["first_token"]
        assert run.completion[i] == q["completion"] and run.restarts[i] == q["restarts"]
    emis = np.concatenate([np.asarray(q["emissions"]) for q in theirs["requests"]])
    assert np.array_equal(run.emissions[:len(emis)], emis)
    rep = run.report_dict()
    for k in ("scheduling_delay", "ttft", "tbt", "e2e", "normalized"):
        for q in ("p50", "p90", "p95", "p99"):
            assert rep[k][q] == theirs["report"][k][q], (k, q)
    assert rep["simulated_span"] == theirs["simulated_span"]
    assert rep["preemptions"] == theirs["report"]["preemptions"]
    timed = ref.simulate_timed(t, cluster, ids, arr, pre, dec)
    assert np.array_equal(timed["completion"], run.completion)


def test_sarathi_chunk_sequence_known_answer(ssg, ref):
    """test_scheduler.cpp:172-191 through the engine: a lone 1300-token prompt under
    Sarathi chunk 512 runs as chunks 512 / 512 / 276 with prior context 0 / 512 /
    1024, then decodes; identical batch log to the reference."""
    m, t = estimators(ssg, ref, "llama2_7b", "a100_80g", [1])
    cluster = catalog.cluster_doc("llama2_7b", "a100_80g", policy="sarathi_serve", max_batch_size=8,
                                  chunk_size=512)
    trace = (np.array([0], dtype=np.int64), np.array([0.0]), np.array([1300], dtype=np.int64),
             np.array([3], dtype=np.int64))
    mine, theirs = run_both(ssg, m, t, cluster, trace)
    assert_same(mine, theirs)
    # entries are [is_prefill, request id, tokens, context]
    chunks = [b["entries"][0] for b in mine["batches"][:3]]
    assert [(e[0], e[2], e[3]) for e in chunks] == [(1, 512, 0), (1, 512, 512), (1, 276, 1024)]
    assert [len(b["entries"]) for b in mine["batches"][3:]] == [1, 1]  # two decodes remain


def test_sarathi_hybrid_batches_fill_the_budget(ssg, ref):
    """test_scheduler.cpp:152-170 as a property of whole runs: decodes are scheduled
    first and a prefill chunk tops the batch up to the 512-token budget whenever a
    long prompt is still being chunked, never beyond it; identical to the reference."""
    m, t = estimators(ssg, ref, "llama2_7b", "a100_80g", [1])
    cluster = catalog.cluster_doc("llama2_7b", "a100_80g", policy="sarathi_serve", max_batch_size=128,
                                  chunk_size=512)
    n = 11
    ids = np.arange(n, dtype=np.int64)
    arr = np.array([i * 0.1 for i in range(10)] + [1.5])
    pre = np.array([1] * 10 + [2000], dtype=np.int64)
    dec = np.array([400] * 10 + [5], dtype=np.int64)  # still decoding at 1.5 s
    mine, theirs = run_both(ssg, m, t, cluster, (ids, arr, pre, dec))
    assert_same(mine, theirs)
    hybrid = 0
    for b in mine["batches"]:
        total = sum(e[2] for e in b["entries"])
        assert total <= 512
        kinds = [e[0] for e in b["entries"]]
        assert kinds == sorted(kinds, reverse=True)  # the log lists prefills, then decodes
        big = [e for e in b["entries"] if e[0] == 1 and e[1] == 10]
        if big and any(e[0] == 0 for e in b["entries"]) and big[0][2] + big[0][3] < 2000:
            assert total == 512  # the chunk fills the budget left by the decodes
            hybrid += 1
    assert hybrid >= 1


@pytest.mark.parametrize("policy,extra", [("vllm", {}), ("orca_plus", {}), ("lightllm", {}),
                                          ("sarathi_serve", {"chunk_size": 256})])
def test_full_batches_with_a_queue(ssg, ref, policy, extra):
    """A lone replica saturated at max_batch_size 16: requests wait while the batch
    is full, which the decode fast-forward treats as a pure-decode stretch (no
    admission can run); identical to the reference."""
    m, t = estimators(ssg, ref, "llama2_7b", "a100_80g", [1])
    cluster = catalog.cluster_doc("llama2_7b", "a100_80g", policy=policy, max_batch_size=16, **extra)
    mine, theirs = run_both(ssg, m, t, cluster, trace_fixture(500, 30.0, 8))
    assert_same(mine, theirs)


@pytest.mark.parametrize("policy,extra", [("vllm", {}), ("orca_plus", {}), ("lightllm", {}),
                                          ("sarathi_serve", {"chunk_size": 256})])
@pytest.mark.parametrize("max_batch,qps", [(8, 40.0), (64, 3.0)])
def test_fast_forward_through_arrivals(ssg, ref, policy, extra, max_batch, qps):
    """Binary-output runs (no batch log) whose decode stretches take arrivals:
    a full batch (max_batch 8, overloaded) keeps its stretch going with a longer
    queue, a batch that is not full (light load) ends it after the iteration the
    request arrives in; the trace tail runs past the last arrival.  Per-request
    times, every token's emission time and the report equal the reference's."""
    m, t = estimators(ssg, ref, "llama2_7b", "a100_80g", [1])
    cluster = catalog.cluster_doc("llama2_7b", "a100_80g", policy=policy, max_batch_size=max_batch, **extra)
    ids, arr, pre, dec = trace_fixture(400, qps, 11)
    run = ssg.simulate_run(cluster, m, ids, arr, pre, dec)
    theirs = t.simulate(cluster, ids, arr, pre, dec)
    for i, q in enumerate(theirs["requests"]):
        assert run.first_scheduled[i] == q["first_scheduled"] and run.first_token[i] == q["first_token"], i
        assert run.completion[i] == q["completion"] and run.restarts[i] == q["restarts"], i
    emis = np.concatenate([np.asarray(q["emissions"]) for q in theirs["requests"]])
    assert np.array_equal(run.emissions[:len(emis)], emis)
    rep = run.report_dict()
    for k in ("scheduling_delay", "ttft", "tbt", "e2e", "normalized"):
        for q in ("p50", "p90", "p95", "p99"):
            assert rep[k][q] == theirs["report"][k][q], (k, q)
    assert rep["simulated_span"] == theirs["simulated_span"]


# acceptance criterion 4 (acceptance.cpp:245-310): LLaMA2-7B on a 30 GB A100,
# 2 round-robin replicas, bs 64 / 4096 tokens / chunk 512, lognormal lengths
# (prefill 300 / 1.0, decode 40 / 0.9, max_total 2048) synth seed 404 at 60 QPS
# seed 405 -- a tight KV pool, so every policy preempts heavily.
ACCEPT4_DEV = dict(catalog.DEVICES["a100_80g"], device_mem=30e9)
ACCEPT4_DIST = {"schema_version": 1, "kind": "lognormal", "prefill": {"median": 300, "sigma": 1.0},
                "decode": {"median": 40, "sigma": 0.9}, "max_total": 2048}


@pytest.mark.slow
@pytest.mark.parametrize("policy", ["faster_transformer", "orca_plus", "vllm", "sarathi_serve",
                                    "lightllm"])
def test_acceptance4_workload(ssg, ref, policy):
    """The reference's scheduler-invariant workload at full size (5 policies x
    10,000 requests): every batch of both replicas, every emission time, the
    aggregates and the report equal the reference's, preemptions included."""
    key = ("accept4",)
    if key not in _EST:
        text = ref.train(catalog.MODELS["llama2_7b"], ACCEPT4_DEV, [1], "interp", 42)
        _EST[key] = (ssg.Estimator.from_json(text), ref.Estimator(text))
    m, t = _EST[key]
    cluster = catalog.cluster_doc("llama2_7b", ACCEPT4_DEV, tp=1, pp=1, replicas=2, policy=policy,
                                  max_batch_size=64, max_tokens_per_iter=4096, chunk_size=512)
    lengths = ssg.synth_trace(ACCEPT4_DIST, 10000, 404)
    mine, theirs = run_both(ssg, m, t, cluster, baseline_trace(ssg, lengths, 60.0, 405))
    assert_same(mine, theirs)
    assert len(theirs["requests"]) == 10000
    if policy == "vllm":  # the policy that preempts to admit (the criterion's 552K preemptions)
        assert sum(r["preemptions"] for r in theirs["replicas"]) > 1000
