"""Multi-GPU sweep plumbing: each rank evaluates its shard of the config grid
(ssg_search_shard / SearchSession.run: a longest-processing-time split on the
configs' initial QPS guesses, identical on every rank), one all-gather of
fixed-size ssg_config_record bytes, finalize on rank 0.

The gather uses whatever torch.distributed backend the caller initialised:
NCCL over NVLink in bench.py, gloo in the CPU tests.  Shards hold different
numbers of configs, so every rank pads its records to the whole grid's count
with index -1 slots; one collective, no size exchange.  Reference: the worker
pool and result vector of run_search (search.hpp:378-393), which this
replaces across GPUs.
"""
from __future__ import annotations

import struct


def live_records(buf: bytes, rec_size: int) -> bytes:
    """Drops the padding slots (index < 0; ssg_config_record.index is the first int64)."""
    out = []
    for off in range(0, len(buf), rec_size):
        if struct.unpack_from("<q", buf, off)[0] >= 0:
            out.append(buf[off: off + rec_size])
    return b"".join(out)


def gather_records(records: bytes, n_configs: int, rank: int, world: int, rec_size: int,
                   device=None) -> bytes:
    """All-gathers each rank's records (padded to n_configs slots); returns
    every rank's records concatenated in rank order."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return records
    assert len(records) % rec_size == 0 and len(records) // rec_size <= n_configs
    pad = torch.zeros(n_configs * rec_size, dtype=torch.uint8)
    pad.view(-1, rec_size)[:, :8] = torch.tensor(list(struct.pack("<q", -1)), dtype=torch.uint8)
    if records:
        pad[: len(records)] = torch.frombuffer(bytearray(records), dtype=torch.uint8)
    buf = pad.to(device) if device is not None else pad
    out = torch.empty(world * n_configs * rec_size, dtype=torch.uint8, device=buf.device)
    dist.all_gather_into_tensor(out, buf)
    return live_records(out.cpu().numpy().tobytes(), rec_size)
