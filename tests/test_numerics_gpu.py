"""Exhaustive check of the device libm (csrc/glibc_math.h on sm_100a) against
the host's glibc over the predictor's whole integer feature domain, in both
glibc contraction variants: the default ifunc mode, and the
SSE2 variant selected with GLIBC_TUNABLES.  ssg_init probes which variant the
host runs and the device reproduces exactly that one -- every log1p input of
the cfg #4/#5 estimators and a dense exp grid must match bit for bit.
reference: estimator.hpp:113-122 (bbox margin, log1p, exp)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = os.path.join(ROOT, "tests", "helpers", "math_domain.py")


def run(env):
    out = subprocess.run([sys.executable, SCRIPT], capture_output=True, text=True, check=True,
                         env=dict(os.environ, **env), timeout=900)
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("mode", ["default", "sse2"])
def test_device_libm_exhaustive_over_feature_domain(mode):
    env = {} if mode == "default" else {"GLIBC_TUNABLES": "glibc.cpu.hwcaps=-AVX2,-FMA"}
    res = run(env)
    if mode == "sse2":
        assert res["variant"] == 0  # the probe saw the SSE2 libm and selected it
    assert res["log1p_values"] > 10_000_000  # the whole domain, not a sample
    for d in res["log1p"]:
        assert d["mismatches"] == 0, d
    assert res["exp"]["mismatches"] == 0, res["exp"]
