"""Drop-in parity of the C++ API (include/servesim_b200.hpp).

tests/cpp/dropin.cpp is ONE caller program -- a cmd_simulate / cmd_search
clone (servesim_cli.cpp:96-178), acceptance criterion 4's invariant observer
(acceptance.cpp:201-310), the scheduler and router known answers of
test_scheduler.cpp, find_capacity / evaluate_config / Regressor calls -- built
twice from the same source: against the reference's headers (oracle/Makefile ->
oracle/_ref/dropin_ref) and against the B200 header + libssg.so (csrc/Makefile
-> build/dropin_ssg).  Every output file and stdout line must be identical.
"""
import filecmp
import os
import subprocess

import numpy as np
import pytest

from paper_2405_05465_b200 import catalog

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SSG_BIN = os.path.join(ROOT, "build", "dropin_ssg")
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_ref")


def run(binary, *args, timeout=900):
    p = subprocess.run([binary, *map(str, args)], capture_output=True, text=True, timeout=timeout)
    return p.returncode, p.stdout, p.stderr


def both(*args, timeout=900):
    if not os.path.exists(REF_BIN):
        pytest.skip("oracle/_ref/dropin_ref not built")
    assert os.path.exists(SSG_BIN), "build/dropin_ssg missing: run __graft_entry__.build()"
    rs = run(SSG_BIN, *args, timeout=timeout)
    rr = run(REF_BIN, *args, timeout=timeout)
    return rs, rr


def test_ref_caller_passes_its_known_answers():
    """CPU: the caller program itself is right (the reference build passes the
    scheduler/router known answers it encodes)."""
    if not os.path.exists(REF_BIN):
        pytest.skip("oracle/_ref/dropin_ref not built")
    rc, out, _ = run(REF_BIN, "scheduler")
    assert rc == 0 and "0 failed" in out.splitlines()[0]


@pytest.mark.gpu
def test_dropin_scheduler_plugin():
    """ReplicaScheduler (GPU-backed) and Router: known answers plus 10 random
    step-by-step traces (5 policies x 2 memory/budget settings, out-of-order
    enqueues, preemptions): every plan, counter and request field identical."""
    (rc, out, err), (rc2, out2, _) = both("scheduler")
    assert rc2 == 0
    assert rc == 0, out[:2000] + err[-2000:]
    assert out.splitlines()[0] == out2.splitlines()[0]
    a, b = out.splitlines(), out2.splitlines()
    for k, (x, y) in enumerate(zip(a, b)):
        assert x == y, "first difference at line %d:\n ssg: %s\n ref: %s" % (k, x, y)
    assert len(a) == len(b)
    assert sum(" pre=" in l and " pre=0 " not in l for l in a) > 50  # preemption paths ran


def _estimator(tmp_path, model, device, tps, regressor="interp", seed=1):
    import paper_2405_05465_b200 as ssg

    est = ssg.Estimator.train(catalog.MODELS[model], catalog.DEVICES[device], list(tps),
                              regressor, seed=seed)
    path = tmp_path / ("est_%s_%s_%s.json" % (model, device, regressor))
    path.write_text(est.to_json())
    return str(path)


SIM_CASES = [
    # (name, cluster kwargs, qps, static, format)
    ("cfg1_vllm_7b", dict(model="llama2_7b", device="a100_80g", policy="vllm", max_batch_size=128), 10.0, 0, "csv"),
    ("sarathi_2rep", dict(model="llama2_7b", device="a100_80g", replicas=2, policy="sarathi_serve",
                          chunk_size=256, max_batch_size=64), 30.0, 0, "json"),
    ("ft_static", dict(model="llama2_7b", device="a100_80g", policy="faster_transformer",
                       max_batch_size=16), 0.0, 1, "csv"),
    ("lo_3rep_pressure", dict(model="llama2_7b", device="a100_80g", replicas=3, policy="vllm",
                              routing="least_outstanding", max_batch_size=48, device_mem=24e9), 40.0, 0, "csv"),
    ("deferred_lightllm", dict(model="llama2_7b", device="a100_80g", replicas=2, policy="lightllm",
                               routing="deferred", max_batch_size=32), 25.0, 0, "json"),
    ("70b_tp2_pp2_orca", dict(model="llama2_70b", device="h100_80g", tp=2, pp=2, policy="orca_plus",
                              max_batch_size=64), 8.0, 0, "csv"),
]


@pytest.mark.gpu
@pytest.mark.parametrize("name,kw,qps,static,fmt", SIM_CASES, ids=[c[0] for c in SIM_CASES])
def test_dropin_cmd_simulate(tmp_path, name, kw, qps, static, fmt):
    """cmd_simulate clone: SimObserver event log (EventLogObserver format,
    servesim_cli.cpp:30-56), requests.csv / requests.json and summary.json are
    byte-identical to the reference's."""
    kw = dict(kw)
    model, device = kw.pop("model"), kw.pop("device")
    tp = kw.get("tp", 1)
    cluster = catalog.write_cluster_config(str(tmp_path / "cfg"), model, device, **kw)
    est = _estimator(tmp_path, model, device, [tp])
    lengths = catalog.fixture_chat_1k()
    trace = catalog.write_trace_csv(str(tmp_path / "trace.csv"), lengths)
    outs = {}
    for tag, binary in (("ssg", SSG_BIN), ("ref", REF_BIN)):
        if not os.path.exists(binary):
            pytest.skip("%s not built" % binary)
        d = tmp_path / tag
        rc, out, err = run(binary, "simulate", cluster, trace, est, d, fmt, qps, 5, static, 1)
        assert rc == 0, (tag, out, err[-2000:])
        outs[tag] = (d, out)
    assert outs["ssg"][1] == outs["ref"][1]
    files = ["events.log", "summary.json", "requests." + fmt]
    for f in files:
        a, b = outs["ssg"][0] / f, outs["ref"][0] / f
        assert a.read_bytes() == b.read_bytes(), f
    assert (outs["ssg"][0] / "events.log").stat().st_size > 1000


@pytest.mark.gpu
def test_dropin_cmd_search(tmp_path):
    """cmd_search clone: results.csv / results.json / both frontiers / summary.txt."""
    cfg = catalog.write_search_config(str(tmp_path / "cfg"), model="llama2_7b", tp=(1, 2), pp=(1, 2),
                                      batch_sizes=(32, 128), chunk_sizes=(512,), probe_requests=400,
                                      num_requests=400, max_gpus_total=8)
    outs = {}
    for tag, binary in (("ssg", SSG_BIN), ("ref", REF_BIN)):
        if not os.path.exists(binary):
            pytest.skip("%s not built" % binary)
        rc, out, err = run(binary, "search", cfg, tmp_path / tag, 3)
        assert rc == 0, (tag, out, err[-2000:])
        outs[tag] = out
    assert outs["ssg"] == outs["ref"]
    for f in ("results.csv", "results.json", "frontier_ttft.csv", "frontier_tbt.csv", "summary.txt"):
        assert filecmp.cmp(tmp_path / "ssg" / f, tmp_path / "ref" / f, shallow=False), f


@pytest.mark.gpu
def test_dropin_acceptance4_invariant_observer(tmp_path):
    """Acceptance criterion 4 through SimOptions::observer: 5 policies x 10K
    requests on 2 round-robin replicas, 30 GB device; zero violations, and the
    observer's per-batch view (tokens, outstanding, preemptions, KV units)
    checksums equal the reference's."""
    d = str(tmp_path)
    model = catalog.write_json(os.path.join(d, "m.json"), catalog.MODELS["llama2_7b"])
    dev = catalog.write_json(os.path.join(d, "d.json"), catalog.DEVICES["a100_80g"])
    (rc, out, err), (rc2, out2, _) = both("invariants", model, dev, timeout=1800)
    assert rc == 0 and rc2 == 0, err[-2000:]
    assert out == out2
    for line in out.splitlines():
        for k in ("mem=0", "batch=0", "tokens=0", "causality=0", "ft=0", "conserve=0", "order=0"):
            assert k in line, line
    assert sum(int(l.split("preemptions=")[1].split()[0]) for l in out.splitlines()) > 1000


@pytest.mark.gpu
def test_dropin_capacity_evaluate_regressor(tmp_path):
    """find_capacity over a callback (same probe sequence), evaluate_config
    (capacity, SLO run, makespan objective, error row), initial_qps_guess, and
    Regressor::predict via regressor_from_json for interp and forest models."""
    d = str(tmp_path)
    model = catalog.write_json(os.path.join(d, "m.json"), catalog.MODELS["llama2_7b"])
    dev = catalog.write_json(os.path.join(d, "d.json"), catalog.DEVICES["a100_80g"])
    (rc, out, err), (rc2, out2, _) = both("capacity", model, dev)
    assert rc == 0 and rc2 == 0, err[-2000:]
    a, b = out.splitlines(), out2.splitlines()
    for x, y in zip(a, b):
        assert x == y
    assert len(a) == len(b)
    assert any("err=estimator: no trained model" in l for l in a)
