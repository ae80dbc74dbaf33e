"""The reference's known-answer vectors (tests/golden/reference_kats.json,
transcribed from /root/reference/proj/tests/*.cpp by
tests/golden/make_reference_kats.py) on the oracle and on the device library."""
import json
from pathlib import Path

import numpy as np
import pytest

from backends import BACKENDS, GroupView, make_backend
from helpers import make_view, rec, records

KATS = json.loads((Path(__file__).parent / "golden" / "reference_kats.json").read_text())


@pytest.fixture(params=BACKENDS)
def be(request):
    return make_backend(request.param)


@pytest.mark.parametrize("k", KATS["split_in_order"], ids=lambda k: k["src"])
def test_split_in_order_kat(be, k):
    v = be.upload(make_view(k["lengths"]))
    g = be.split_in_order(v, k["B"], k["order"])
    assert [list(x.col("length")) for x in g] == k["group_lengths"]
    assert [list(x.col("skip")) for x in g] == k["group_skips"]
    assert [x.total_steps for x in g] == k["group_steps"]


@pytest.mark.parametrize("k", KATS["pack_batch_sizes"], ids=lambda k: k["src"])
def test_pack_batch_sizes_kat(be, k):
    hv = make_view(k["lengths"])
    b = be.pack(be.upload(hv), GroupView(hv.seqs, hv.size))
    assert list(b.batch_sizes) == k["batch_sizes"]


@pytest.mark.parametrize("k", KATS["gae"], ids=lambda k: k["src"])
def test_gae_kat(be, k):
    hv = make_view(k["lengths"])
    hv.reward[:] = k["reward"]
    hv.value[:] = k["value"]
    if k["done"] is not None:
        hv.done[:] = k["done"]
    if k["bootstrap_valid"] is not None:
        hv.env_bootstrap_valid[0] = k["bootstrap_valid"]
    v = be.upload(hv)
    be.gae(v, k["gamma"], k["lambda"])
    a = be.host(v).advantage
    if "advantage" in k:
        assert np.allclose(a, k["advantage"], atol=1e-6)
    else:
        assert a[k["check_index"]] == pytest.approx(k["check_advantage"])


@pytest.mark.parametrize("k", KATS["estimate_time"], ids=lambda k: k["src"])
def test_estimate_time_kat(be, k):
    for s, t in zip(k["steps"], k["time"]):
        assert be.estimate_time(k["tau"], k["max_steps"], s) == pytest.approx(t, abs=1e-12)


@pytest.mark.parametrize("k", KATS["optimal_preempt_steps"], ids=lambda k: k["src"])
def test_optimal_preempt_kat(be, k):
    assert be.optimal_preempt_steps(k["tau"], k["learn_time"], k["max_steps"]) == k["s_star"]


@pytest.mark.parametrize("k", KATS["sequence_lengths"], ids=lambda k: k["src"])
def test_sequence_lengths_kat(be, k):
    buf = be.rollout(k["T"], k["N"], 1)
    buf.begin_rollout(1)
    buf.append(records([rec(e, ep, t, bool(d)) for e, ep, t, d in k["records"]]))
    v = be.host(buf.close_rollout())
    assert list(v.seqs[:, 2]) == k["seq_lengths"]
