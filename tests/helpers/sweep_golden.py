"""Sweep goldens (tests/golden/sweep): the compiled reference's run_search
outputs for whole config grids, made by tools/make_sweep_golden.py.  Shared by
the generator, the GPU parity test and bench.py."""
import hashlib
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
GOLDEN = os.path.join(ROOT, "tests", "golden", "sweep")
FILES = (("results_csv", "results.csv"), ("frontier_ttft_csv", "frontier_ttft.csv"),
         ("frontier_tbt_csv", "frontier_tbt.csv"), ("summary", "summary.txt"))

# case -> catalog.write_search_config arguments (SURVEY.md 8(d) cfg #4 / #5)
CASES = {
    "cfg4": dict(model="llama2_70b", workload="chat_like"),
    "cfg5_qwen72b_arxiv": dict(model="qwen_72b", workload="arxiv_like"),
    "cfg5_internlm20b_bwb": dict(model="internlm_20b", workload="bwb_like"),
}


def config_digest(path: str) -> str:
    """sha256 over the search document and every document beside it."""
    h = hashlib.sha256()
    base = os.path.dirname(path)
    for root, _, files in sorted(os.walk(base)):
        for f in sorted(files):
            p = os.path.join(root, f)
            h.update(os.path.relpath(p, base).encode())
            with open(p, "rb") as fh:
                h.update(fh.read())
    return h.hexdigest()


def load(case: str, variant: str):
    """(outputs dict, meta dict) or None when the golden is absent."""
    d = os.path.join(GOLDEN, "%s.%s" % (case, variant))
    if not os.path.isdir(d):
        return None
    out = {}
    for k, f in FILES:
        with open(os.path.join(d, f)) as fh:
            out[k] = fh.read()
    with open(os.path.join(d, "meta.json")) as fh:
        return out, json.load(fh)
