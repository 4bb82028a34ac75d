"""Multi-GPU sweep plumbing: configs i % world == rank per process, one
all-gather of fixed-size ssg_config_record bytes, finalize on rank 0.

The gather uses whatever torch.distributed backend the caller initialised:
NCCL over NVLink in bench.py, gloo in the CPU tests.  Reference: the worker
pool and result vector of run_search (search.hpp:378-393), which this
replaces across GPUs.
"""
from __future__ import annotations


def shard_sizes(n_configs: int, world: int):
    return [len(range(r, n_configs, world)) for r in range(world)]


def gather_records(records: bytes, n_configs: int, rank: int, world: int, rec_size: int,
                   device=None) -> bytes:
    """All-gathers each rank's records (padded to the largest shard); returns
    every rank's records concatenated in rank order."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return records
    per_rank = -(-n_configs // world)
    buf = torch.zeros(per_rank * rec_size, dtype=torch.uint8, device=device)
    if records:
        buf[: len(records)] = torch.frombuffer(bytearray(records), dtype=torch.uint8).to(buf.device)
    out = torch.empty(world * per_rank * rec_size, dtype=torch.uint8, device=device)
    dist.all_gather_into_tensor(out, buf)
    host = out.cpu().numpy().tobytes()
    sizes = shard_sizes(n_configs, world)
    return b"".join(host[r * per_rank * rec_size: r * per_rank * rec_size + sizes[r] * rec_size]
                    for r in range(world))
