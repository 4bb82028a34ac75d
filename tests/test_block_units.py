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
