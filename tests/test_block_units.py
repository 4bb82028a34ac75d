"""CPU: the device's block count ceil(t / b) = mulhi(t + b - 1, block_magic(b))
(engine.cuh units_for, sim_device.h block_magic) over every block size a
config can carry up to 4096 and every token count the engine can reach for
it, plus the power-of-two and large-size edges.  The GPU parity tests cover
block sizes 1, 7, 24 and 32 end to end (test_engine_gpu.py::test_block_sizes)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = r'''
#include <cstdio>
#include <cstdint>
#include <initializer_list>
#include "sim_device.h"
static int64_t units(int64_t t, int64_t b, bool tg) {
  const uint64_t m = block_magic(b, tg);
  return m ? (int64_t)(((unsigned __int128)(uint64_t)(t + b - 1) * m) >> 64) : t;
}
int main() {
  long bad = 0, n = 0;
  for (int64_t b = 1; b <= 4096; ++b) {
    const int64_t step = b < 64 ? 1 : 97;
    for (int64_t t = 0; t < (int64_t(1) << 20); t += step, ++n)
      if (units(t, b, false) != (t + b - 1) / b) ++bad;
    for (int64_t t = (int64_t(1) << 31) - 4096; t < (int64_t(1) << 31); ++t, ++n)
      if (units(t, b, false) != (t + b - 1) / b) ++bad;
  }
  for (int k = 0; k < 31; ++k) {
    const int64_t b = int64_t(1) << k;
    for (int64_t t : {int64_t(0), int64_t(1), b - 1, b, b + 1, (int64_t(1) << 31) - 1}) {
      ++n;
      if (units(t, b, false) != (t + b - 1) / b) ++bad;
    }
  }
  for (int64_t b : {int64_t(3), int64_t(1000003), (int64_t(1) << 31) - 1})
    for (int64_t t = 0; t < (int64_t(1) << 31); t += (int64_t(1) << 31) / 4099, ++n)
      if (units(t, b, false) != (t + b - 1) / b) ++bad;
  for (int64_t t = 0; t < 100000; ++t, ++n)
    if (units(t, 16, true) != t) ++bad;  // LightLLM: one unit per token
  std::printf("%ld %ld\n", bad, n);
  return bad != 0;
}
'''


def test_block_magic_is_exact(tmp_path):
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("no host C++ compiler")
    src = tmp_path / "units.cpp"
    src.write_text(SRC)
    exe = tmp_path / "units"
    subprocess.run([gxx, "-O2", "-std=c++17", "-I", os.path.join(ROOT, "paper_2405_05465_b200", "csrc"),
                    str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    bad, n = map(int, out.stdout.split())
    assert bad == 0 and n > 10_000_000, out.stdout


def _units(x, b):
    return -(-x // b)


def _closed_form_needs(kv, held, done, kir, b):
    """engine.cu fast_forward_t's block needs of one runner over iterations
    done .. done+kir-1: units(kv+1) - held at k = 0 (if positive), then one
    block exactly at the k >= 1 where kv + k is a multiple of b and
    kv + k >= held * b; the remainder uses floor(x / b) = mulhi(x, magic)."""
    got = [0] * kir
    if done == 0:
        got[0] += max(0, _units(kv + 1, b) - held)
    kmin = max(max(1, done), held * b - kv)
    x = kv + kmin
    m = _magic(b)
    rr = x - ((x * m) >> 64) * b
    k = kmin if rr == 0 else kmin + (b - rr)
    while k < done + kir:
        got[k - done] += 1
        k += b
    return got


def _magic(b):
    if b & (b - 1) == 0:
        return 1 << (64 - (b.bit_length() - 1))
    return (1 << 64) // b + 1


@pytest.mark.parametrize("b", [2, 3, 7, 16, 24, 32, 48])
def test_fast_forward_closed_form_block_needs(b):
    """The closed form equals the per-iteration definition the event loop
    applies (reserve kv+k+1 tokens holding max(held, units(kv+k)) for k >= 1),
    for every context, high-water mark and round start in range."""
    for kv in range(0, 5 * b + 3):
        for held in range(0, _units(kv, b) + 3):
            for done in (0, 1, 2, b - 1, b, 3 * b + 1):
                kir = 32
                ref = []
                for i in range(kir):
                    k = done + i
                    hk = held if k == 0 else max(held, _units(kv + k, b))
                    ref.append(max(0, _units(kv + k + 1, b) - hk))
                assert _closed_form_needs(kv, held, done, kir, b) == ref, (kv, held, done)
