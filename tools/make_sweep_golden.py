"""Generates the Vidur-Search sweep goldens (tests/golden/sweep/) from the
compiled REFERENCE (oracle/_ref): load_search_config + run_search + the three
writers (config.hpp:111-179, search.hpp:369-486), run with workers = nproc.

Run in the build container (needs /root/reference compiled by `make -C oracle`):
    python tools/make_sweep_golden.py [case ...]
Cases:
  cfg4                 the bench's cfg #4 grid: LLaMA2-70B x chat_like, 450 configs,
                       2000 probe requests, tol 0.02, interp (catalog defaults)
  cfg5_qwen72b_arxiv   cfg #5 pair Qwen-72B x arxiv_like (450 configs)
  cfg5_internlm20b_bwb cfg #5 pair InternLM-20B x bwb_like (450 configs)
Each case is recorded under BOTH glibc libm contraction variants: the default
(FMA on this host) and the SSE2 variant in a child process with
GLIBC_TUNABLES=glibc.cpu.hwcaps=-AVX2,-FMA.  Output per case and variant:
  tests/golden/sweep/<case>.<fma|plain>/{results.csv, frontier_ttft.csv,
                                         frontier_tbt.csv, summary.txt, meta.json}
meta.json pins the sha256 of the search-config document the case was run on,
so a change to catalog.write_search_config invalidates the golden loudly.
"""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2405_05465_b200 import catalog  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "tests", "helpers"))
from sweep_golden import CASES, FILES, GOLDEN as OUT, config_digest  # noqa: E402


def run_case(name: str, variant: str):
    d = tempfile.mkdtemp(prefix="sweep_golden_")
    path = catalog.write_search_config(d, **CASES[name])
    workers = os.cpu_count() or 1
    out = ref.search(path, workers=workers)
    dst = os.path.join(OUT, "%s.%s" % (name, variant))
    os.makedirs(dst, exist_ok=True)
    for key, fn in FILES:
        with open(os.path.join(dst, fn), "w") as f:
            f.write(out[key])
    meta = {"case": name, "variant": variant, "config_sha256": config_digest(path),
            "configs": out["configs"], "seconds": out["seconds"], "workers": workers,
            "args": CASES[name],
            "generator": "tools/make_sweep_golden.py (reference compiled by oracle/Makefile)"}
    with open(os.path.join(dst, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("%-22s %-5s %d configs in %.1f s" % (name, variant, out["configs"], out["seconds"]),
          flush=True)


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--child":
        return run_case(sys.argv[2], "plain")
    names = sys.argv[1:] or list(CASES)
    for n in names:
        run_case(n, "fma")  # this container's libm is the FMA variant
        env = dict(os.environ, GLIBC_TUNABLES="glibc.cpu.hwcaps=-AVX2,-FMA")
        subprocess.run([sys.executable, __file__, "--child", n], env=env, check=True)


if __name__ == "__main__":
    main()
