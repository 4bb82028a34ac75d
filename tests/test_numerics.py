"""glibc-exact exp/log1p (csrc/glibc_math.h) against this host's libm, in the
default ifunc mode and -- via GLIBC_TUNABLES -- the non-FMA SSE2 mode.
The same header is compiled into the sm_100a kernels (--fmad=false), so this
pins the device arithmetic on the CPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def harness(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("num") / "numerics_check")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-I",
                    os.path.join(ROOT, "paper_2405_05465_b200", "csrc"),
                    os.path.join(ROOT, "tests", "helpers", "numerics_check.c"), "-lm", "-o", exe],
                   check=True)
    return exe


def run(exe, env=None, n=2_000_000):
    out = subprocess.run([exe, str(n)], capture_output=True, text=True, check=True,
                         env=dict(os.environ, **(env or {}))).stdout.split()
    return [int(v) for v in out]  # plain exp, plain log1p, fma exp, fma log1p


def test_default_libm_matches_one_variant_exactly(harness):
    pe, pl, fe, fl = run(harness)
    assert (pe, pl) == (0, 0) or (fe, fl) == (0, 0)
    assert (pe + pl) != (fe + fl)  # the variants really differ on these inputs


def test_non_fma_libm_matches_plain_variant(harness):
    pe, pl, fe, fl = run(harness, {"GLIBC_TUNABLES": "glibc.cpu.hwcaps=-AVX2,-FMA"})
    assert (pe, pl) == (0, 0)


def test_library_probe_agrees():
    from paper_2405_05465_b200 import math_variant

    assert math_variant() in (0, 1)
