"""Model, device and workload catalog for the BASELINE configurations.

The reference ships these as JSON documents under proj/configs/; the same
facts are kept here as Python data and rendered to JSON on demand, so a search
or cluster document can be written anywhere (tests use tmp dirs) and both the
GPU path and the oracle read byte-identical inputs.

Sources (reference, read-only):
  models   proj/configs/models/{llama2_7b,llama2_70b,internlm_20b,qwen_72b}.json
  devices  proj/configs/devices/{a100_80g,h100_80g}.json
  traces   proj/configs/workloads/{chat_like,bwb_like}.json; arxiv_like is
           derived as SURVEY.md §8(d) prescribes (Arxiv-4K
           prefill median 2730, decode median 167; sigma = ln(p90/median)/1.2816)
  fixture  proj/fixtures/traces/synthetic_chat_1k.csv -> tests/golden/chat_1k_lengths.npy
"""
from __future__ import annotations

import json
import os

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _model(name, layers, hidden, q, kv, head, mlp, vocab, variant):
    return {
        "schema_version": 1, "name": name, "num_layers": layers, "hidden_dim": hidden,
        "num_q_heads": q, "num_kv_heads": kv, "head_dim": head, "mlp_dim": mlp,
        "vocab_size": vocab, "max_context": 4096, "param_bytes_per_element": 2,
        "attention_variant": variant,
    }


MODELS = {
    "llama2_7b": _model("llama2-7b", 32, 4096, 32, 32, 128, 11008, 32000, "mha"),
    "llama2_70b": _model("llama2-70b", 80, 8192, 64, 8, 128, 28672, 32000, "gqa"),
    "internlm_20b": _model("internlm-20b", 60, 5120, 40, 40, 128, 13824, 103168, "mha"),
    "qwen_72b": _model("qwen-72b", 80, 8192, 64, 64, 128, 24576, 152064, "mha"),
}

DEVICES = {
    "a100_80g": {"schema_version": 1, "sku_name": "A100-80G", "peak_flops": 312e12,
                 "mem_bandwidth": 2.039e12, "link_bandwidth": 3.0e11,
                 "kernel_overhead": 2e-6, "device_mem": 80e9},
    "h100_80g": {"schema_version": 1, "sku_name": "H100-80G", "peak_flops": 989e12,
                 "mem_bandwidth": 3.35e12, "link_bandwidth": 4.5e11,
                 "kernel_overhead": 2e-6, "device_mem": 80e9},
}

COST_TABLE = {"A100-80G": 2.5, "H100-80G": 4.2}


def _lognormal(pm, ps, dm, ds):
    return {"schema_version": 1, "kind": "lognormal",
            "prefill": {"median": pm, "sigma": ps}, "decode": {"median": dm, "sigma": ds},
            "max_total": 4096}


WORKLOADS = {
    "chat_like": _lognormal(417, 1.086, 139, 0.973),
    "bwb_like": _lognormal(1037, 0.263, 1601, 0.230),
    "arxiv_like": _lognormal(2730, 0.238, 167, 0.625),
}


def zipf_histogram(exponent: float = 1.1, max_total: int = 4096) -> dict:
    """SURVEY.md §8(d) cfg #2: prefill min(4095, 32k), decode 8j, weight k^-a j^-a."""
    bins = []
    for k in range(1, 129):
        for j in range(1, 65):
            bins.append({"prefill": min(4095, 32 * k), "decode": 8 * j,
                         "weight": (k ** -exponent) * (j ** -exponent)})
    return {"schema_version": 1, "kind": "histogram", "bins": bins, "max_total": max_total}


def fixture_chat_1k():
    """The reference's bundled 1000-request fixture: (prefill, decode) pairs, ids 0..999."""
    import numpy as np

    return np.load(os.path.join(_ROOT, "tests", "golden", "chat_1k_lengths.npy"))


def write_json(path: str, doc) -> str:
    os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
    return path


def cluster_doc(model: str, device: str, tp=1, pp=1, replicas=1, policy="vllm",
                routing="round_robin", cpu_overhead=0.0, **sched) -> dict:
    """Inline cluster document (model spec and device embedded)."""
    scheduler = {"policy": policy}
    scheduler.update(sched)
    return {
        "model_spec": MODELS[model] if isinstance(model, str) else model,
        "device": DEVICES[device] if isinstance(device, str) else device,
        "parallelism": {"tp_degree": tp, "pp_degree": pp, "num_replicas": replicas},
        "scheduler": scheduler,
        "routing": {"policy": routing},
        "cpu_overhead_per_iter": cpu_overhead,
    }


def write_search_config(directory: str, model: str = "llama2_70b", workload: str = "chat_like",
                        skus=("a100_80g", "h100_80g"), tp=(1, 2, 4), pp=(1, 2, 4),
                        schedulers=("vllm", "orca_plus", "sarathi_serve"),
                        batch_sizes=(32, 64, 128, 256, 512), chunk_sizes=(512, 1024, 2048),
                        max_gpus_total=16, num_requests=2000, synth_seed=7,
                        probe_requests=2000, tolerance=0.02, objective="qps_per_dollar",
                        workload_doc=None, device_docs=None) -> str:
    """Renders a reference-format search config (config.hpp:111-179) plus the
    model/device documents it points at; returns the config path.
    `device_docs` adds SKUs beyond DEVICES ({key: device document}; their
    hourly rate is 1.0)."""
    os.makedirs(directory, exist_ok=True)
    devices = dict(DEVICES, **(device_docs or {}))
    write_json(os.path.join(directory, "models", model + ".json"), MODELS[model])
    for s in skus:
        write_json(os.path.join(directory, "devices", s + ".json"), devices[s])
    cfg = {
        "schema_version": 1,
        "model_spec": "models/%s.json" % model,
        "workload": {"synthetic": workload_doc or WORKLOADS[workload],
                     "num_requests": num_requests, "synth_seed": synth_seed},
        "space": {"skus": ["devices/%s.json" % s for s in skus], "tp_degrees": list(tp),
                  "pp_degrees": list(pp), "schedulers": list(schedulers),
                  "batch_sizes": list(batch_sizes), "chunk_sizes": list(chunk_sizes),
                  "max_gpus_total": max_gpus_total},
        "slos": {"ttft_p90_max": 2.0, "tbt_p99_max": 0.2, "delay_p99_max": 5.0},
        "cost_table": {devices[s]["sku_name"]: COST_TABLE.get(devices[s]["sku_name"], 1.0)
                       for s in skus},
        "capacity": {"tolerance": tolerance, "probe_requests": probe_requests,
                     "evaluation_fraction": 0.85},
        "objective": objective,
    }
    return write_json(os.path.join(directory, "search.json"), cfg)


def write_cluster_config(directory: str, model: str, device: str, tp=1, pp=1, replicas=1,
                         policy="vllm", routing="round_robin", cpu_overhead=0.0,
                         device_mem=None, **sched) -> str:
    """File-form cluster config (config.hpp:71-98): model and device documents
    beside it, referenced by relative path; returns the config path."""
    os.makedirs(directory, exist_ok=True)
    dev = dict(DEVICES[device])
    if device_mem is not None:
        dev["device_mem"] = device_mem
    write_json(os.path.join(directory, "models", model + ".json"), MODELS[model])
    write_json(os.path.join(directory, "devices", device + ".json"), dev)
    scheduler = {"policy": policy}
    scheduler.update(sched)
    cfg = {"schema_version": 1, "model_spec": "models/%s.json" % model,
           "device": "devices/%s.json" % device,
           "parallelism": {"tp_degree": tp, "pp_degree": pp, "num_replicas": replicas},
           "scheduler": scheduler, "routing": {"policy": routing},
           "cpu_overhead_per_iter": cpu_overhead}
    return write_json(os.path.join(directory, "cluster.json"), cfg)


def write_trace_csv(path: str, lengths, arrivals=None) -> str:
    """Reference trace CSV (workload.hpp:28-79): ids 0..n-1, with or without arrivals."""
    os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
    with open(path, "w") as f:
        if arrivals is None:
            f.write("request_id,prefill_tokens,decode_tokens\n")
            for i, (p, d) in enumerate(lengths):
                f.write("%d,%d,%d\n" % (i, p, d))
        else:
            f.write("request_id,arrival_time_s,prefill_tokens,decode_tokens\n")
            for i, ((p, d), a) in enumerate(zip(lengths, arrivals)):
                f.write("%d,%r,%d,%d\n" % (i, float(a), p, d))
    return path
