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
