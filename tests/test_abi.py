"""C ABI surface (CPU-only): the library loads, exports every ssg.h entry
point, and fails loudly (status 3, no fallback) when no GPU is present."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "ssg.h")).read()
    return sorted(set(re.findall(r"\b(ssg_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2405_05465_b200 import _ffi

    lib = _ffi.lib()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert len(declared_symbols()) >= 12


def test_python_binding_covers_header():
    from paper_2405_05465_b200 import _ffi

    assert set(declared_symbols()) <= set(_ffi.exported_symbols())


def test_no_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2405_05465_b200 as ssg

    with pytest.raises(ssg.CudaError):
        ssg.init(0)


def test_host_training_without_gpu():
    """Training is host work (profiling + fitting); it must not need the device."""
    import json

    import paper_2405_05465_b200 as ssg
    from paper_2405_05465_b200 import catalog

    est = ssg.Estimator.train(catalog.MODELS["llama2_7b"], catalog.DEVICES["a100_80g"], [1], "interp", 1)
    doc = json.loads(est.to_json())
    assert doc["kind"] == "estimator" and "attn_decode@tp1" in doc["ops"]
