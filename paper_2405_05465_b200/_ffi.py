"""ctypes binding of libssg.so (include/ssg.h).

The library is built in-tree (`make -C paper_2405_05465_b200/csrc`, or
`__graft_entry__.build()`); importing this module without it raises -- there
is no Python or CPU fallback for any compute entry point.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SSG_LIB: an alternative build of the same library (A/B experiments only)
LIB_PATH = os.environ.get("SSG_LIB") or os.path.join(_HERE, "libssg.so")

OK, INPUT, INTERNAL, CUDA = 0, 1, 2, 3


class Status(C.Structure):
    _fields_ = [("code", C.c_int32), ("message", C.c_char * 4096)]


class SsgError(RuntimeError):
    """Base of the library's errors; `.code` is the ssg.h status."""

    code = INTERNAL


class InputError(SsgError):
    """servesim::Error -- the message is the reference's verbatim."""

    code = INPUT


class InternalError(SsgError):
    code = INTERNAL


class CudaError(SsgError):
    code = CUDA


_ERRORS = {INPUT: InputError, INTERNAL: InternalError, CUDA: CudaError}

_lib = None

P = C.c_void_p
pd = C.POINTER(C.c_double)
pi64 = C.POINTER(C.c_int64)
pi32 = C.POINTER(C.c_int32)

_SIGNATURES = {
    "ssg_init": (C.c_int, [C.c_int, C.POINTER(Status)]),
    "ssg_shutdown": (C.c_int, []),
    "ssg_math_variant": (C.c_int, []),
    "ssg_math_check": (C.c_int, [C.c_int, C.c_double, C.c_double, C.c_int64, pi64, pd,
                                 C.POINTER(Status)]),
    "ssg_version": (C.c_char_p, []),
    "ssg_free": (None, [P]),
    "ssg_estimator_from_json": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(P), C.POINTER(Status)]),
    "ssg_estimator_train": (C.c_int, [C.c_char_p, C.c_char_p, pi64, C.c_size_t, C.c_char_p,
                                      C.c_uint64, C.POINTER(P), C.POINTER(Status)]),
    "ssg_estimator_to_json": (C.c_int, [P, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t),
                                        C.POINTER(Status)]),
    "ssg_estimator_free": (None, [P]),
    "ssg_estimator_slot": (C.c_int32, [P, C.c_int32, C.c_int64]),
    "ssg_estimator_device_bytes": (C.c_int64, [P, C.POINTER(Status)]),
    "ssg_predict": (C.c_int, [P, C.c_int32, C.c_int64, C.c_size_t, P, P, P, C.POINTER(Status)]),
    "ssg_predict_mixed": (C.c_int, [P, C.c_size_t, P, P, P, P, C.POINTER(Status)]),
    "ssg_predict_device": (C.c_int, [P, C.c_size_t, P, C.c_int32, P, P, P, P, P,
                                     C.POINTER(Status)]),
    "ssg_predict_batch": (C.c_int, [P, C.c_char_p, C.c_int64, C.c_size_t, P, P, P, P, P, P, P,
                                    C.POINTER(Status)]),
    "ssg_synth_trace": (C.c_int, [C.c_char_p, C.c_size_t, C.c_uint64, P, P, C.POINTER(Status)]),
    "ssg_poisson_arrivals": (C.c_int, [C.c_size_t, C.c_double, C.c_uint64, P, C.POINTER(Status)]),
    "ssg_cap_total_length": (C.c_int, [C.c_size_t, P, P, C.c_int64, C.POINTER(Status)]),
    "ssg_load_trace": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(Status)]),
    "ssg_simulate_run": (C.c_int, [C.c_char_p, P, C.c_size_t, P, P, P, P, C.c_int, P, P, P, P, P,
                                   P, C.POINTER(Status)]),
    "ssg_simulate": (C.c_int, [C.c_char_p, P, C.c_size_t, P, P, P, P, C.c_int, C.c_double,
                               C.c_size_t, C.c_int, C.POINTER(C.c_void_p), C.POINTER(Status)]),
    "ssg_search": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_void_p),
                             C.POINTER(Status)]),
    "ssg_search_shard": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_void_p, C.c_size_t,
                                   C.POINTER(C.c_size_t), C.POINTER(Status)]),
    "ssg_search_finalize": (C.c_int, [C.c_char_p, P, C.c_size_t, C.POINTER(C.c_void_p),
                                      C.POINTER(Status)]),
    "ssg_search_record_size": (C.c_size_t, []),
    "ssg_search_open": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(Status)]),
    "ssg_search_run": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_size_t,
                                 C.POINTER(C.c_size_t), C.POINTER(Status)]),
    "ssg_search_num_configs": (C.c_int64, [C.c_void_p]),
    "ssg_search_close": (None, [C.c_void_p]),
    "ssg_stats_reset": (None, []),
    "ssg_stats_get": (None, [C.c_void_p]),
}


def lib():
    """Loads libssg.so once; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            "libssg.so not built (%s); run `make -C paper_2405_05465_b200/csrc` "
            "or __graft_entry__.build()" % LIB_PATH)
    L = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(L, name, None)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


class RunStats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "launches_simulate", "launches_select", "launches_predict", "launches_batch", "units",
        "iterations", "entries", "events", "predictor_bytes", "entry_bytes", "queries")] + [
        ("simulate_ms", C.c_double), ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
        ("launches_setup", C.c_int64), ("simulate_busy_ms", C.c_double),
        ("useful_iterations", C.c_int64), ("useful_entries", C.c_int64), ("useful_bytes", C.c_int64),
        ("cancelled_probes", C.c_int64), ("spec_slo_runs", C.c_int64), ("spec_slo_used", C.c_int64)]


def exported_symbols():
    return list(_SIGNATURES)


def check(rc: int, st: Status):
    if rc != OK:
        raise _ERRORS.get(rc, SsgError)(st.message.decode("utf-8", "replace"))


def call(name, *args):
    st = Status()
    rc = getattr(lib(), name)(*args, C.byref(st))
    check(rc, st)
    return rc


def take_text(ptr: C.c_void_p) -> str:
    """Copies and frees a NUL-terminated buffer returned by the library."""
    if not ptr.value:
        return ""
    s = C.string_at(ptr.value).decode("utf-8")
    lib().ssg_free(ptr)
    return s


class MetricSummary(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("mean", "p50", "p90", "p95", "p99")]


class SimReport(C.Structure):
    _fields_ = ([("simulated_span", C.c_double), ("total_model_flops", C.c_double),
                 ("num_devices", C.c_int64)]
                + [(n, MetricSummary) for n in ("scheduling_delay", "ttft", "tbt", "e2e", "normalized")]
                + [("mfu", C.c_double), ("kv_utilization_peak", C.c_double),
                   ("busy_fraction", C.c_double), ("preemptions", C.c_int64)])
