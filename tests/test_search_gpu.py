"""Vidur-Search parity: the GPU sweep vs the compiled reference run_search.

results.csv, both frontier CSVs and summary.txt must be byte-identical --
capacities (exact doubles from the replayed find_capacity), SLO percentiles
(exact selections), ranking and the chosen optimum.
reference: search.hpp:369-486, config.hpp:111-179.
"""
import os

import pytest

from paper_2405_05465_b200 import catalog

pytestmark = pytest.mark.gpu


def compare(mine, theirs):
    assert mine["results_csv"] == theirs["results_csv"]
    assert mine["frontier_ttft_csv"] == theirs["frontier_ttft_csv"]
    assert mine["frontier_tbt_csv"] == theirs["frontier_tbt_csv"]
    assert mine["summary"] == theirs["summary"]


def test_search_7b_example(ssg, ref, tmp_path):
    """The reference's own example search (configs/search/llama2_7b_example.json shape)."""
    path = catalog.write_search_config(
        str(tmp_path), model="llama2_7b", skus=("a100_80g", "h100_80g"), tp=(1,), pp=(1,),
        schedulers=("vllm", "sarathi_serve"), batch_sizes=(32, 128), chunk_sizes=(512,),
        max_gpus_total=8, num_requests=2000, probe_requests=2000)
    compare(ssg.search(path), ref.search(path, workers=os.cpu_count() or 1))


def test_search_70b_slice_all_policies(ssg, ref, tmp_path):
    """cfg #4 slice: LLaMA2-70B, both SKUs, TP/PP mix, the three searched schedulers."""
    path = catalog.write_search_config(
        str(tmp_path), model="llama2_70b", tp=(2, 4), pp=(1, 2), batch_sizes=(64, 256),
        chunk_sizes=(512, 2048), probe_requests=1000, num_requests=1000)
    compare(ssg.search(path), ref.search(path, workers=os.cpu_count() or 1))


def test_search_makespan_objective(ssg, ref, tmp_path):
    path = catalog.write_search_config(
        str(tmp_path), model="llama2_7b", skus=("a100_80g",), tp=(1, 2), pp=(1,),
        schedulers=("vllm", "orca_plus", "sarathi_serve"), batch_sizes=(32, 128),
        chunk_sizes=(512,), max_gpus_total=4, probe_requests=500, num_requests=500,
        objective="makespan")
    compare(ssg.search(path), ref.search(path, workers=os.cpu_count() or 1))


def test_search_error_rows(ssg, ref, tmp_path):
    """TP1 70B does not fit an 80 GB device: "insufficient device memory" rows."""
    path = catalog.write_search_config(
        str(tmp_path), model="llama2_70b", skus=("a100_80g",), tp=(1, 4), pp=(1,),
        schedulers=("vllm",), batch_sizes=(128,), probe_requests=600, num_requests=600)
    mine, theirs = ssg.search(path), ref.search(path, workers=2)
    compare(mine, theirs)
    assert "insufficient device memory" in mine["results_csv"]


def test_sharded_search_equals_whole(ssg, tmp_path):
    """Shards evaluated separately and finalized together == the one-GPU outcome
    (the multi-GPU path: each rank a shard, records all-gathered)."""
    path = catalog.write_search_config(
        str(tmp_path), model="llama2_7b", skus=("a100_80g", "h100_80g"), tp=(1, 2), pp=(1,),
        schedulers=("vllm", "sarathi_serve"), batch_sizes=(32, 128), chunk_sizes=(512,),
        max_gpus_total=8, probe_requests=800, num_requests=800)
    whole = ssg.search(path)
    recs = b"".join(ssg.search_shard(path, s, 3) for s in range(3))
    compare(ssg.search_finalize(path, recs), whole)


def test_concurrent_sessions_equal_sequential(ssg, tmp_path):
    """Sweeps run on several host threads at once (the cfg #5 bench does this):
    each session borrows its own streams and buffers, and every session's records
    are byte-identical to running them one after another."""
    from concurrent.futures import ThreadPoolExecutor

    paths = [catalog.write_search_config(
        str(tmp_path / ("s%d" % i)), model=m, workload=w, skus=("a100_80g",), tp=(1, 2), pp=(1, 2),
        schedulers=("vllm", "sarathi_serve", "orca_plus"), batch_sizes=(32, 128), chunk_sizes=(512,),
        max_gpus_total=8, probe_requests=600, num_requests=600)
        for i, (m, w) in enumerate([("llama2_7b", "chat_like"), ("llama2_70b", "bwb_like"),
                                    ("qwen_72b", "arxiv_like")])]
    sessions = [ssg.SearchSession(p) for p in paths]
    sequential = [s.run() for s in sessions]
    with ThreadPoolExecutor(len(sessions)) as ex:
        concurrent = list(ex.map(lambda s: s.run(), sessions))
    for a, b in zip(sequential, concurrent):
        assert a == b
    with ThreadPoolExecutor(len(paths)) as ex:  # one-call form, fresh sessions per thread
        fresh = list(ex.map(lambda p: ssg.search_shard(p, 0, 1), paths))
    for a, b in zip(sequential, fresh):
        assert a == b
    for s in sessions:
        s.close()


def _golden_case(ssg, case, tmp_path):
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "helpers"))
    import sweep_golden

    variant = "fma" if ssg.math_variant() == 1 else "plain"
    g = sweep_golden.load(case, variant)
    if g is None:
        pytest.skip("no %s golden for libm variant %s" % (case, variant))
    theirs, meta = g
    path = catalog.write_search_config(str(tmp_path), **sweep_golden.CASES[case])
    # the grid this run evaluates is the one the reference evaluated
    assert sweep_golden.config_digest(path) == meta["config_sha256"]
    return path, theirs


@pytest.mark.slow
@pytest.mark.parametrize("case", ["cfg4", "cfg5_qwen72b_arxiv", "cfg5_internlm20b_bwb"])
def test_full_grid_matches_reference(ssg, case, tmp_path):
    """The headline sweeps, whole grids (450 configs, 2000 probe requests each):
    cfg #4 (LLaMA2-70B x chat_like) and two cfg #5 pairs (Qwen-72B x arxiv_like,
    InternLM-20B x bwb_like), byte-identical to the reference's own run_search
    outputs (tests/golden/sweep, tools/make_sweep_golden.py) -- every capacity,
    percentile, error row, the ranking, both frontiers and the chosen optimum."""
    path, theirs = _golden_case(ssg, case, tmp_path)
    compare(ssg.search(path), theirs)


@pytest.mark.slow
@pytest.mark.parametrize("shards", [2, 8])
def test_full_grid_sharded_matches_reference(ssg, shards, tmp_path):
    """cfg #4 split over `shards` ranks by the cost-based (LPT) assignment, each
    shard evaluated on its own, records merged: the same bytes as the reference."""
    path, theirs = _golden_case(ssg, "cfg4", tmp_path)
    parts = [ssg.search_shard(path, s, shards) for s in range(shards)]
    size = ssg.record_size()
    assert sum(len(p) for p in parts) == 450 * size  # the shards partition the grid
    compare(ssg.search_finalize(path, b"".join(parts)), theirs)


# A 7B replica on this device holds ~1,500 KV tokens (params 10.59 GB + 10 %
# reserve), so the chat_like trace's longer requests cannot be served.
TINY_GPU = {"schema_version": 1, "sku_name": "TINY-GPU", "peak_flops": 312e12,
            "mem_bandwidth": 2.039e12, "link_bandwidth": 3.0e11, "kernel_overhead": 2e-6,
            "device_mem": 12.64e9}


@pytest.mark.parametrize("objective", ["makespan", "qps_per_dollar"])
def test_search_oversized_requests_two_replicas(ssg, ref, tmp_path, objective):
    """Requests beyond a replica's KV capacity raise from enqueue on both
    round-robin replicas.  Under the makespan objective every arrival is at
    t = 0, so the two replicas fail at the same clock: the error row must name
    the request the reference meets first in its (time, seq) event order
    (scheduler.hpp:146-155; sim.hpp:211-220), not the first replica's."""
    path = catalog.write_search_config(
        str(tmp_path), model="llama2_7b", skus=("tiny",), tp=(1,), pp=(1,),
        schedulers=("vllm", "sarathi_serve"), batch_sizes=(32,), chunk_sizes=(512,),
        max_gpus_total=2, probe_requests=400, num_requests=400, objective=objective,
        device_docs={"tiny": TINY_GPU})
    mine, theirs = ssg.search(path), ref.search(path, workers=2)
    compare(mine, theirs)
    assert "KV units but replica capacity" in mine["results_csv"]

# ~3,000 KV tokens per 7B replica: only the trace's rare longest requests are
# oversized, so whether a probe raises depends on its rate (a fast probe can
# abort on late schedules before the first oversized request arrives).
SMALL_GPU = dict(TINY_GPU, sku_name="SMALL-GPU", device_mem=13.51e9)


def test_search_deep_speculation_same_answers(ssg, ref, tmp_path, monkeypatch):
    """Speculation never changes an answer: with an 8-rate doubling ladder and
    bisection sub-trees 6 levels deep, rates the sequential find_capacity never
    asks are simulated too -- including rates whose probes raise -- and the
    outcome is still the reference's (probe errors are memoised and surface
    only when the replay asks for that rate; search.hpp:145-174)."""
    monkeypatch.setenv("SSG_SPEC_LADDER", "8")
    monkeypatch.setenv("SSG_SPEC_DEPTH", "6")
    path = catalog.write_search_config(
        str(tmp_path), model="llama2_7b", skus=("a100_80g", "small"), tp=(1, 2), pp=(1,),
        schedulers=("vllm", "orca_plus", "sarathi_serve"), batch_sizes=(32, 256),
        chunk_sizes=(512,), max_gpus_total=4, probe_requests=600, num_requests=600,
        device_docs={"small": SMALL_GPU})
    compare(ssg.search(path), ref.search(path, workers=os.cpu_count() or 1))


@pytest.mark.slow
@pytest.mark.parametrize("knobs", [
    # every under-loaded rule forced on for the whole grid: speculative SLO runs at
    # every capacity a settling round can end with, lag depth, a six-rung ladder and
    # bisection sub-trees under every ladder bracket
    {"SSG_SPEC_SLO": "8", "SSG_SPEC_LAG": "2", "SSG_SPEC_LADDER": "6", "SSG_SPEC_PRE": "2"},
    # and every one forced off, on one lane
    {"SSG_SPEC_SLO": "0", "SSG_SPEC_LAG": "0", "SSG_SPEC_LADDER": "4", "SSG_SPEC_PRE": "0",
     "SSG_LANES": "1"},
])
def test_full_grid_speculation_rules_same_answers(ssg, knobs, tmp_path, monkeypatch):
    """The sweep's scheduling rules (search.cpp SweepKnobs: which rates and SLO runs a
    round speculates, how many candidate lanes) only move work between rounds: cfg #4
    under either extreme is byte-identical to the reference's run_search."""
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    path, theirs = _golden_case(ssg, "cfg4", tmp_path)
    compare(ssg.search(path), theirs)
