"""Workload generation parity: the host-side inputs that
feed every simulation and capacity probe -- synth_trace (lognormal and
histogram), poisson_arrivals, cap_total_length and load_trace -- against the
compiled reference (workload.hpp:33-247), bit for bit, including the error
messages.  CPU only: these are the host half of the path."""
import numpy as np
import pytest

import paper_2405_05465_b200 as ssg
from paper_2405_05465_b200 import catalog
from paper_2405_05465_b200._ffi import SsgError


def same_error(ref, mine, theirs):
    with pytest.raises(SsgError) as a:
        mine()
    with pytest.raises(ref.RefError) as b:
        theirs()
    assert str(a.value) == str(b.value)


@pytest.mark.parametrize("name", ["chat_like", "bwb_like", "arxiv_like"])
@pytest.mark.parametrize("seed", [0, 7, 42])
def test_synth_lognormal(ref, name, seed):
    dist = catalog.WORKLOADS[name]
    pre, dec = ssg.synth_trace(dist, 5000, seed)
    want = ref.workload("synth", dist=dist, n=5000, seed=seed)
    assert np.array_equal(pre, want["prefill"]) and np.array_equal(dec, want["decode"])
    assert want["id"] == list(range(5000))


def test_synth_zipf_histogram_cfg2(ref):
    """cfg #2's 10K Zipf trace: identical draws, and the summary
    statistics the survey quotes for it (prefill mean 627 / median 192 / p90 2016,
    decode mean 94 / median 40 / p90 288)."""
    dist = catalog.zipf_histogram()
    pre, dec = ssg.synth_trace(dist, 10000, 42)
    want = ref.workload("synth", dist=dist, n=10000, seed=42)
    assert np.array_equal(pre, want["prefill"]) and np.array_equal(dec, want["decode"])

    def nearest_rank(v, q):
        s = np.sort(v)
        return s[int(np.ceil(q * len(s))) - 1]

    assert round(pre.mean()) == 627 and nearest_rank(pre, 0.5) == 192 and nearest_rank(pre, 0.9) == 2016
    assert round(dec.mean()) == 94 and nearest_rank(dec, 0.5) == 40 and nearest_rank(dec, 0.9) == 288


def test_synth_capped_and_small(ref):
    dist = dict(catalog.WORKLOADS["bwb_like"], max_total=2)
    pre, dec = ssg.synth_trace(dist, 300, 3)
    want = ref.workload("synth", dist=dist, n=300, seed=3)
    assert np.array_equal(pre, want["prefill"]) and np.array_equal(dec, want["decode"])
    assert ssg.synth_trace(dist, 0, 3)[0].size == 0


@pytest.mark.parametrize("rate", [0.3, 5.0, 10.0, 20.0, 1e6, 1e13])
@pytest.mark.parametrize("seed", [0, 1, 5])
def test_poisson_arrivals(ref, rate, seed):
    got = ssg.poisson_arrivals(10000, rate, seed)
    want = ref.workload("poisson", n=10000, rate=rate, seed=seed)["arrivals"]
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    assert np.all(np.diff(got) > 0)


def test_cap_total_length(ref):
    rng = np.random.default_rng(0)
    pre = rng.integers(1, 9000, 4000)
    dec = rng.integers(1, 9000, 4000)
    for m in (2, 3, 512, 4096, 20000):
        a = ssg.cap_total_length(pre, dec, m)
        b = ref.workload("cap", prefill=pre.tolist(), decode=dec.tolist(), max_total=m)
        assert np.array_equal(a[0], b["prefill"]) and np.array_equal(a[1], b["decode"]), m
        assert np.all(a[0] + a[1] <= m) and np.all(a[0] >= 1) and np.all(a[1] >= 1)


def test_workload_errors(ref):
    same_error(ref, lambda: ssg.cap_total_length([5], [5], 1),
               lambda: ref.workload("cap", prefill=[5], decode=[5], max_total=1))
    same_error(ref, lambda: ssg.poisson_arrivals(3, 0.0, 1),
               lambda: ref.workload("poisson", n=3, rate=0.0, seed=1))
    bad = [dict(catalog.WORKLOADS["chat_like"], kind="gamma"),
           dict(catalog.WORKLOADS["chat_like"], schema_version=2),
           {"schema_version": 1, "kind": "lognormal", "prefill": {"median": 5, "sigma": -1},
            "decode": {"median": 5, "sigma": 1}},
           {"schema_version": 1, "kind": "histogram", "bins": []},
           {"schema_version": 1, "kind": "histogram", "bins": [{"prefill": 0, "decode": 1, "weight": 1}]},
           {"schema_version": 1, "kind": "histogram", "bins": [{"prefill": 3, "decode": 1, "weight": 0}]},
           {"schema_version": 1, "kind": "lognormal", "prefill": {"median": 5}}]
    for d in bad:
        same_error(ref, lambda: ssg.synth_trace(d, 4, 1), lambda: ref.workload("synth", dist=d, n=4, seed=1))


def trace_csv(with_arrival: bool, n=200, crlf=False, seed=0):
    lengths = catalog.fixture_chat_1k()[:n]
    rng = np.random.default_rng(seed)
    arr = np.round(rng.random(n) * 50, 3)  # unsorted, with ties
    arr[5] = arr[9]
    eol = "\r\n" if crlf else "\n"
    if with_arrival:
        lines = ["request_id,arrival_time_s,prefill_tokens,decode_tokens"]
        lines += ["%d,%r,%d,%d" % (i, float(a), p, d) for i, (a, (p, d)) in enumerate(zip(arr, lengths))]
    else:
        lines = ["request_id,prefill_tokens,decode_tokens"]
        lines += ["%d,%d,%d" % (i, p, d) for i, (p, d) in enumerate(lengths)]
    return eol.join(lines) + eol


@pytest.mark.parametrize("with_arrival", [True, False])
@pytest.mark.parametrize("crlf", [False, True])
def test_load_trace(ref, with_arrival, crlf):
    text = trace_csv(with_arrival, crlf=crlf)
    got = ssg.load_trace(text)
    want = ref.workload("load_trace", text=text)
    for k in ("id", "prefill", "decode"):
        assert np.array_equal(got[k], want[k]), k
    if with_arrival:
        assert np.array_equal(got["arrival"].view(np.uint64), want["arrival"].view(np.uint64))
    else:
        assert got["arrival"] is None and want["arrival"] is None


def test_load_trace_errors(ref):
    cases = ["", "id,prefill,decode\n1,2,3\n",
             "request_id,prefill_tokens,decode_tokens\n1,2\n",
             "request_id,prefill_tokens,decode_tokens\n1,x,3\n",
             "request_id,prefill_tokens,decode_tokens\n1,2,0\n",
             "request_id,arrival_time_s,prefill_tokens,decode_tokens\n1,-1,2,3\n",
             "request_id,arrival_time_s,prefill_tokens,decode_tokens\n1,abc,2,3\n",
             "request_id,prefill_tokens,decode_tokens\n1.5,2,3\n"]
    for text in cases:
        same_error(ref, lambda: ssg.load_trace(text), lambda: ref.workload("load_trace", text=text))
