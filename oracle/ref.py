"""TEST INFRASTRUCTURE: ctypes handle on the compiled reference (oracle/_ref).

`make -C oracle` builds oracle/_ref/libservesim_ref.so from the unmodified
reference headers under /root/reference (see oracle/Makefile).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.environ.get("SSG_REF_LIB", os.path.join(HERE, "_ref", "libservesim_ref.so"))

_lib = None

P = C.c_void_p


def available() -> bool:
    return os.path.exists(LIB)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise ImportError("oracle not built: %s (run `make -C oracle`)" % LIB)
        L = C.CDLL(LIB)
        L.ref_free.argtypes = [P]
        for name, args in {
            "ref_train": [C.c_char_p, C.c_char_p, P, C.c_size_t, C.c_char_p, C.c_uint64],
            "ref_predict_batch": [P, C.c_char_p, C.c_int64, C.c_size_t, P, P, P, P, P, P, P],
            "ref_simulate": [C.c_char_p, P, C.c_size_t, P, P, P, P, C.c_int, C.c_double,
                             C.c_size_t, C.c_int],
            "ref_search": [C.c_char_p, C.c_int],
            "ref_evaluate_sample": [C.c_char_p, P, C.c_size_t, C.c_int],
            "ref_workload": [C.c_char_p],
            "ref_simulate_timed": [C.c_char_p, P, C.c_size_t, P, P, P, P],
        }.items():
            fn = getattr(L, name)
            fn.restype = C.c_void_p
            fn.argtypes = args
        L.ref_estimator_load.restype = P
        L.ref_estimator_load.argtypes = [C.c_char_p]
        L.ref_estimator_free.argtypes = [P]
        L.ref_predict.restype = C.c_long
        L.ref_predict.argtypes = [P, P, P, C.c_size_t, P, P, P, C.c_char_p, C.c_size_t]
        L.ref_predict_timed.restype = C.c_double
        L.ref_predict_timed.argtypes = [P, P, P, C.c_size_t, P, P, P, C.c_int]
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, kind, msg):
        super().__init__(msg)
        self.kind = kind


def _raw(ptr) -> str:
    s = C.string_at(ptr).decode()
    lib().ref_free(ptr)
    return s


def _text(ptr) -> dict:
    j = json.loads(_raw(ptr))
    if isinstance(j, dict) and "error" in j and "kind" in j:
        raise RefError(j["kind"], j["error"])
    return j


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def train(model_spec: dict, device: dict, tps, regressor="interp", seed=0) -> str:
    arr = np.asarray(tps, dtype=np.int64)
    ptr = lib().ref_train(json.dumps(model_spec).encode(), json.dumps(device).encode(), _p(arr),
                          len(arr), regressor.encode(), seed)
    text = _raw(ptr)  # the reference's own nlohmann dump, byte for byte
    j = json.loads(text)
    if "error" in j and "kind" in j:
        raise RefError(j["kind"], j["error"])
    return text


class Estimator:
    def __init__(self, est_json: str):
        self.h = lib().ref_estimator_load(est_json.encode())
        if not self.h:
            raise RefError("Error", "oracle could not load estimator json")

    def __del__(self):
        try:
            lib().ref_estimator_free(self.h)
        except Exception:
            pass

    def predict(self, ops, tps, f0, f1=None):
        """Returns (out, first_failing_index or -1, message)."""
        n = len(f0)
        ops = np.ascontiguousarray(np.broadcast_to(ops, (n,)), dtype=np.int32)
        tps = np.ascontiguousarray(np.broadcast_to(tps, (n,)), dtype=np.int64)
        f0 = np.ascontiguousarray(f0, dtype=np.float64)
        f1 = np.zeros(n) if f1 is None else np.ascontiguousarray(f1, dtype=np.float64)
        out = np.zeros(n)
        err = C.create_string_buffer(4096)
        bad = lib().ref_predict(self.h, _p(ops), _p(tps), n, _p(f0), _p(f1), _p(out), err, 4096)
        return out, int(bad), err.value.decode()

    def predict_timed(self, ops, tps, f0, f1, threads):
        n = len(f0)
        ops = np.ascontiguousarray(ops, dtype=np.int32)
        tps = np.ascontiguousarray(tps, dtype=np.int64)
        f0 = np.ascontiguousarray(f0, dtype=np.float64)
        f1 = np.ascontiguousarray(f1, dtype=np.float64)
        out = np.zeros(n)
        secs = lib().ref_predict_timed(self.h, _p(ops), _p(tps), n, _p(f0), _p(f1), _p(out), threads)
        return out, secs

    def predict_batch(self, model_spec: dict, tp: int, batches):
        p_off, p_len, p_prior, d_off, d_ctx = [0], [], [], [0], []
        for pl, pp, dc in batches:
            p_len += list(pl)
            p_prior += list(pp)
            d_ctx += list(dc)
            p_off.append(len(p_len))
            d_off.append(len(d_ctx))
        arrs = [np.asarray(a, dtype=np.int64) for a in (p_off, p_len, p_prior, d_off, d_ctx)]
        secs = np.zeros(len(batches))
        flops = np.zeros(len(batches))
        res = _text(lib().ref_predict_batch(self.h, json.dumps(model_spec).encode(), tp, len(batches),
                                            *[_p(a) for a in arrs], _p(secs), _p(flops)))
        return secs, flops, res

    def simulate(self, cluster: dict, ids, arrivals, prefill, decode, record_batches=False,
                 abort_delay=0.0, abort_max_late=0, static_mode=False) -> dict:
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        arr = np.ascontiguousarray(arrivals, dtype=np.float64)
        pre = np.ascontiguousarray(prefill, dtype=np.int64)
        dec = np.ascontiguousarray(decode, dtype=np.int64)
        return _text(lib().ref_simulate(json.dumps(cluster).encode(), self.h, len(ids), _p(ids),
                                        _p(arr), _p(pre), _p(dec), int(record_batches),
                                        abort_delay, abort_max_late, int(static_mode)))


def simulate_timed(est: "Estimator", cluster: dict, ids, arrivals, prefill, decode) -> dict:
    """run_simulation + build_report on one thread, timed inside the reference build."""
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    arr = np.ascontiguousarray(arrivals, dtype=np.float64)
    pre = np.ascontiguousarray(prefill, dtype=np.int64)
    dec = np.ascontiguousarray(decode, dtype=np.int64)
    j = _text(lib().ref_simulate_timed(json.dumps(cluster).encode(), est.h, len(ids), _p(ids),
                                       _p(arr), _p(pre), _p(dec)))
    j["completion"] = np.array(j.pop("completion_bits"), dtype=np.uint64).view(np.float64)
    return j


def search(config_path: str, workers: int = 1) -> dict:
    return _text(lib().ref_search(config_path.encode(), workers))


def evaluate_sample(config_path: str, indices, workers: int) -> dict:
    idx = np.ascontiguousarray(indices, dtype=np.int64)
    return _text(lib().ref_evaluate_sample(config_path.encode(), _p(idx), len(idx), workers))


def workload(op: str, **kw) -> dict:
    """synth_trace / poisson_arrivals / cap_total_length / load_trace of the
    reference (workload.hpp:33-247).  Doubles come back as float64 arrays."""
    kw["op"] = op
    j = _text(lib().ref_workload(json.dumps(kw).encode()))
    for k in ("arrivals", "arrival"):
        if j.get(k) is not None:
            j[k] = np.array(j[k], dtype=np.uint64).view(np.float64)
    return j
