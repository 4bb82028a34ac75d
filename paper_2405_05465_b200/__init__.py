"""B200-native servesim hot path: predictor, replica simulation, capacity search.

Python is the test/bench harness only; every call below goes through the C
ABI in include/ssg.h into libssg.so (sm_100a kernels + host C++).  See
DESIGN.md for the architecture and INTEGRATION.md for the reference-side
bindings.
"""
from __future__ import annotations

import ctypes as C
import json
from typing import Optional, Sequence

import numpy as np

from . import _ffi
from ._ffi import CudaError, InputError, InternalError, SsgError

OPS = ["qkv_proj", "attn_out_proj", "mlp_up_proj", "mlp_down_proj", "act_fn", "add_norm",
       "attn_prefill", "attn_decode", "allreduce", "allgather", "send_recv"]
OP_INDEX = {n: i for i, n in enumerate(OPS)}

__all__ = ["init", "Estimator", "OPS", "OP_INDEX", "SsgError", "InputError", "InternalError",
           "CudaError", "math_variant", "simulate", "search"]


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def init(device: int = 0) -> None:
    """Selects the GPU (ssg_init); also probes the host libm variant."""
    _ffi.call("ssg_init", device)


def math_variant() -> int:
    return _ffi.lib().ssg_math_variant()


def math_check(fn: str, base: float, step: float, n: int):
    """Device log1p / exp (the glibc restatement, host variant) at base + k*step,
    k in [0, n), against this host's libm: (mismatches, first mismatching x)."""
    bad = C.c_int64(0)
    first = C.c_double(0.0)
    _ffi.call("ssg_math_check", {"log1p": 0, "exp": 1}[fn], float(base), float(step), int(n),
              C.byref(bad), C.byref(first))
    return bad.value, first.value


class Estimator:
    """Trained per-operator predictors (reference EstimatorModel, estimator.hpp:90-181)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    @classmethod
    def from_json(cls, text: str) -> "Estimator":
        h = C.c_void_p()
        b = text.encode()
        _ffi.call("ssg_estimator_from_json", b, len(b), C.byref(h))
        return cls(h)

    @classmethod
    def train(cls, model_spec: dict, device: dict, tps: Sequence[int], regressor: str = "interp",
              seed: int = 0) -> "Estimator":
        h = C.c_void_p()
        arr = np.asarray(tps, dtype=np.int64)
        _ffi.call("ssg_estimator_train", json.dumps(model_spec).encode(), json.dumps(device).encode(),
                  arr.ctypes.data_as(_ffi.pi64), len(arr), regressor.encode(), seed, C.byref(h))
        return cls(h)

    def to_json(self) -> str:
        out = C.c_void_p()
        n = C.c_size_t()
        _ffi.call("ssg_estimator_to_json", self._h, C.byref(out), C.byref(n))
        return _ffi.take_text(out)

    @property
    def handle(self):
        return self._h

    def slot(self, op: str, tp: int) -> int:
        return _ffi.lib().ssg_estimator_slot(self._h, OP_INDEX[op], tp)

    def device_bytes(self) -> int:
        st = _ffi.Status()
        n = _ffi.lib().ssg_estimator_device_bytes(self._h, C.byref(st))
        _ffi.check(st.code, st)
        return n

    def predict(self, op: str, tp: int, f0, f1=None) -> np.ndarray:
        """EstimatorModel::predict over arrays of features (host buffers)."""
        f0 = np.ascontiguousarray(f0, dtype=np.float64)
        f1 = None if f1 is None else np.ascontiguousarray(f1, dtype=np.float64)
        out = np.empty_like(f0)
        _ffi.call("ssg_predict", self._h, OP_INDEX[op], tp, len(f0), _ptr(f0), _ptr(f1), _ptr(out))
        return out

    def predict_mixed(self, slots, f0, f1=None, out=None) -> np.ndarray:
        slots = np.ascontiguousarray(slots, dtype=np.int32)
        f0 = np.ascontiguousarray(f0, dtype=np.float64)
        f1 = None if f1 is None else np.ascontiguousarray(f1, dtype=np.float64)
        if out is None:
            out = np.empty_like(f0)
        _ffi.call("ssg_predict_mixed", self._h, len(f0), _ptr(slots), _ptr(f0), _ptr(f1), _ptr(out))
        return out

    def predict_device(self, n: int, slots_ptr: int, uniform_slot: int, f0_ptr: int, f1_ptr: int,
                       out_ptr: int, err_ptr: int, stream: int = 0) -> None:
        """Device-pointer form (e.g. torch tensors' data_ptr()), enqueued on `stream`."""
        _ffi.call("ssg_predict_device", self._h, n, slots_ptr or None, uniform_slot, f0_ptr,
                  f1_ptr or None, out_ptr, err_ptr, stream or None)

    def predict_batch(self, model_spec: dict, tp: int, batches):
        """predict_batch + batch_device_flops over compositions
        [(prefill_lengths, prefill_priors, decode_contexts), ...]."""
        p_off, p_len, p_prior, d_off, d_ctx = [0], [], [], [0], []
        for pl, pp, dc in batches:
            p_len += list(pl)
            p_prior += list(pp)
            d_ctx += list(dc)
            p_off.append(len(p_len))
            d_off.append(len(d_ctx))
        arrs = [np.asarray(a, dtype=np.int64) for a in (p_off, p_len, p_prior, d_off, d_ctx)]
        secs = np.empty(len(batches))
        flops = np.empty(len(batches))
        _ffi.call("ssg_predict_batch", self._h, json.dumps(model_spec).encode(), tp, len(batches),
                  *[_ptr(a) for a in arrs], _ptr(secs), _ptr(flops))
        return secs, flops

    def __del__(self):
        try:
            if self._h:
                _ffi.lib().ssg_estimator_free(self._h)
                self._h = None
        except Exception:
            pass


def synth_trace(dist: dict, n: int, seed: int):
    """synth_trace (workload.hpp:213-247): (prefill, decode) int64 arrays of n requests."""
    pre = np.zeros(n, dtype=np.int64)
    dec = np.zeros(n, dtype=np.int64)
    _ffi.call("ssg_synth_trace", json.dumps(dist).encode(), n, seed, _ptr(pre), _ptr(dec))
    return pre, dec


def poisson_arrivals(n: int, rate_qps: float, seed: int) -> np.ndarray:
    """poisson_arrivals (workload.hpp:93-104): arrival times of n requests."""
    out = np.zeros(n, dtype=np.float64)
    _ffi.call("ssg_poisson_arrivals", n, rate_qps, seed, _ptr(out))
    return out


def cap_total_length(prefill, decode, max_total: int):
    """cap_total_length (workload.hpp:109-121): capped copies of the lengths."""
    pre = np.array(prefill, dtype=np.int64)
    dec = np.array(decode, dtype=np.int64)
    _ffi.call("ssg_cap_total_length", len(pre), _ptr(pre), _ptr(dec), max_total)
    return pre, dec


def load_trace(csv_text: str) -> dict:
    """load_trace (workload.hpp:33-78): {"id", "arrival" (or None), "prefill", "decode"}."""
    out = C.c_void_p()
    _ffi.call("ssg_load_trace", csv_text.encode(), C.byref(out))
    j = json.loads(_ffi.take_text(out))
    return {k: (None if j[k] is None else np.array(j[k])) for k in ("id", "arrival", "prefill", "decode")}


class SimulationRun:
    """Binary outputs of ssg_simulate_run: per-request arrays in trace order, the
    emission times (CSR by decode length), and the report."""

    def __init__(self, n: int, total_decode: int, pinned=None):
        alloc = pinned or (lambda k, dt: np.empty(k, dtype=dt))
        self.first_scheduled = alloc(n, np.float64)
        self.first_token = alloc(n, np.float64)
        self.completion = alloc(n, np.float64)
        self.restarts = alloc(n, np.int64)
        self.emissions = alloc(max(1, total_decode), np.float64)
        self.report = _ffi.SimReport()

    def report_dict(self) -> dict:
        r = self.report
        out = {k: getattr(r, k) for k in ("simulated_span", "total_model_flops", "num_devices", "mfu",
                                          "kv_utilization_peak", "busy_fraction", "preemptions")}
        for k in ("scheduling_delay", "ttft", "tbt", "e2e", "normalized"):
            m = getattr(r, k)
            out[k] = {q: getattr(m, q) for q in ("mean", "p50", "p90", "p95", "p99")}
        return out


def simulate_run(cluster: dict, estimator: Estimator, ids, arrivals, prefill, decode,
                 static_mode: bool = False, out: Optional[SimulationRun] = None) -> SimulationRun:
    """run_simulation + build_report through ssg_simulate_run (binary outputs)."""
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    arr = np.ascontiguousarray(arrivals, dtype=np.float64)
    pre = np.ascontiguousarray(prefill, dtype=np.int64)
    dec = np.ascontiguousarray(decode, dtype=np.int64)
    if out is None:
        out = SimulationRun(len(ids), int(dec.sum()))
    _ffi.call("ssg_simulate_run", json.dumps(cluster).encode(), estimator.handle, len(ids), _ptr(ids),
              _ptr(arr), _ptr(pre), _ptr(dec), int(static_mode), _ptr(out.first_scheduled),
              _ptr(out.first_token), _ptr(out.completion), _ptr(out.restarts), _ptr(out.emissions),
              C.byref(out.report))
    return out


def simulate(cluster: dict, estimator: Estimator, ids, arrivals, prefill, decode,
             record_batches: bool = False, abort_delay: float = 0.0, abort_max_late: int = 0,
             static_mode: bool = False) -> dict:
    """run_simulation + build_report through ssg_simulate (sim.hpp:135-320)."""
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    arr = np.ascontiguousarray(arrivals, dtype=np.float64)
    pre = np.ascontiguousarray(prefill, dtype=np.int64)
    dec = np.ascontiguousarray(decode, dtype=np.int64)
    out = C.c_void_p()
    _ffi.call("ssg_simulate", json.dumps(cluster).encode(), estimator.handle, len(ids), _ptr(ids),
              _ptr(arr), _ptr(pre), _ptr(dec), int(record_batches), abort_delay, abort_max_late,
              int(static_mode), C.byref(out))
    return json.loads(_ffi.take_text(out))


def search(config_path: str) -> dict:
    """run_search from a reference-format search config (config.hpp:111, search.hpp:369)."""
    out = C.c_void_p()
    _ffi.call("ssg_search", config_path.encode(), 0, 1, C.byref(out))
    return json.loads(_ffi.take_text(out))


def record_size() -> int:
    return _ffi.lib().ssg_search_record_size()


def search_shard(config_path: str, shard: int, num_shards: int) -> bytes:
    """This shard's ConfigResults as fixed-size records (ssg_config_record), for all-gather."""
    import math

    # capacity: every config could land in one shard (a search is at most a few
    # thousand configs; the library reports an error if the buffer is short)
    cap = 1 << 14
    size = record_size()
    buf = (C.c_char * (cap * size))()
    n = C.c_size_t()
    _ffi.call("ssg_search_shard", config_path.encode(), shard, num_shards, buf, cap, C.byref(n))
    return bytes(buf[: n.value * size])


def search_finalize(config_path: str, records: bytes) -> dict:
    """Ranking + Pareto + writers over all shards' records."""
    size = record_size()
    assert len(records) % size == 0
    out = C.c_void_p()
    buf = C.create_string_buffer(records, len(records))
    _ffi.call("ssg_search_finalize", config_path.encode(), buf, len(records) // size, C.byref(out))
    return json.loads(_ffi.take_text(out))


class SearchSession:
    """A prepared sweep (ssg_search_open): estimators resident in HBM; run() is the hot path."""

    def __init__(self, config_path: str):
        self._h = C.c_void_p()
        self.path = config_path
        _ffi.call("ssg_search_open", config_path.encode(), C.byref(self._h))
        self.num_configs = _ffi.lib().ssg_search_num_configs(self._h)

    def run(self, shard: int = 0, num_shards: int = 1) -> bytes:
        size = record_size()
        cap = self.num_configs
        buf = (C.c_char * (cap * size))()
        n = C.c_size_t()
        _ffi.call("ssg_search_run", self._h, shard, num_shards, buf, cap, C.byref(n))
        return bytes(buf[: n.value * size])

    def close(self):
        if self._h:
            _ffi.lib().ssg_search_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def stats_reset() -> None:
    _ffi.lib().ssg_stats_reset()


def stats() -> dict:
    s = _ffi.RunStats()
    _ffi.lib().ssg_stats_get(C.byref(s))
    return {name: getattr(s, name) for name, _ in s._fields_}


def decode_records(records: bytes) -> list:
    """Fixed-size ssg_config_record bytes -> dicts (for inspection / tests)."""
    size = record_size()
    out = []
    for k in range(0, len(records), size):
        r = records[k:k + size]
        idx = int.from_bytes(r[0:8], "little", signed=True)
        vals = np.frombuffer(r[8:56], dtype=np.float64)
        slo = int.from_bytes(r[56:60], "little", signed=True)
        err = r[64:].split(b"\0", 1)[0].decode()
        out.append(dict(index=idx, capacity_qps=vals[0], qps_per_dollar=vals[1], ttft_p90=vals[2],
                        tbt_p99=vals[3], delay_p99=vals[4], makespan=vals[5], slo_pass=bool(slo),
                        error=err))
    return out
