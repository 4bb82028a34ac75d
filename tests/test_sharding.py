"""Multi-process host logic of the sharded sweep (CPU, gloo, world size 2):
records of each rank's configs are all-gathered and finalized; the outcome
equals finalizing all records in one process (ranking/Pareto/writers are
order-independent of the shard split; shards may be uneven).  The GPU evaluation itself is covered
by tests/test_search_gpu.py::test_sharded_search_equals_whole."""
import os
import struct
import tempfile

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def fake_record(index, rec_size):
    # ssg_config_record: index, 6 doubles, slo_pass, reserved, error[960]
    cap = 10.0 + (index * 7919 % 97) / 3.0
    err = b"" if index % 11 else b"insufficient device memory: test"
    if err:
        cap = 0.0
    body = struct.pack("<q6dii", index, cap, cap / 40.0, 0.5 + index % 5 / 10.0,
                       0.05 + index % 7 / 100.0, 1.0, 0.0, int(index % 3 != 0), 0)
    return (body + err).ljust(rec_size, b"\0")


def worker(rank, world, cfg_path, port, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_2405_05465_b200 as ssg
    from paper_2405_05465_b200.shard import gather_records

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 16
        size = ssg.record_size()
        # uneven shards, as the cost-based (LPT) split produces: rank 0 holds 11
        # configs, rank 1 the other 5, in no particular index order
        split = [[15, 0, 2, 3, 4, 6, 7, 9, 10, 12, 13], [14, 1, 5, 8, 11]]
        mine = b"".join(fake_record(i, size) for i in split[rank])
        allrecs = gather_records(mine, n, rank, world, size)
        if rank == 0:
            q.put(ssg.search_finalize(cfg_path, allrecs))
    finally:
        dist.destroy_process_group()


def test_two_rank_gather_finalize():
    import paper_2405_05465_b200 as ssg
    from paper_2405_05465_b200 import catalog

    d = tempfile.mkdtemp()
    cfg = catalog.write_search_config(d, model="llama2_7b", skus=("a100_80g", "h100_80g"),
                                      tp=(1, 2), pp=(1,), schedulers=("vllm", "sarathi_serve"),
                                      batch_sizes=(32, 128), chunk_sizes=(512,), max_gpus_total=8)
    size = ssg.record_size()
    whole = ssg.search_finalize(cfg, b"".join(fake_record(i, size) for i in range(16)))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=worker, args=(r, 2, cfg, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == whole
    assert "insufficient device memory: test" in got["results_csv"]
    assert got["configs"] == 16
