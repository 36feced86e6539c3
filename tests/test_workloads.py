"""The host workload generator against the reference's own arrays
(tests/golden/workloads.json, made by tests/golden/make_workloads.py from
the real sparsekv): every array bit-identical, same needle positions."""

import hashlib
import json
import os

import numpy as np
import pytest

from paper_2502_14866_b200 import workloads as W


def _fixture(golden_dir):
    with open(os.path.join(golden_dir, "workloads.json")) as fp:
        return json.load(fp)


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, np.float64).tobytes()).hexdigest()


def test_gen_workload_bit_identical_to_reference(golden_dir):
    for rec in _fixture(golden_dir)["specs"]:
        w, t = W.gen_workload(W.WorkloadSpec(**rec["spec"]))
        assert (digest(w.q), digest(w.k), digest(w.v)) == (rec["q"], rec["k"], rec["v"]), rec["spec"]
        assert list(t.needle_positions) == rec["positions"]
        assert list(t.needle_pages) == rec["pages"]


def test_spec_validation():
    with pytest.raises(ValueError, match="unknown workload kind"):
        W.WorkloadSpec(kind="haystack")
    with pytest.raises(ValueError, match="multiple"):
        W.WorkloadSpec(num_heads=3, num_kv_heads=2)
    with pytest.raises(ValueError, match="no full page"):
        W.gen_workload(W.WorkloadSpec(kind="needle", num_history=40))
    with pytest.raises(ValueError, match="margin"):
        W.gen_workload(W.WorkloadSpec(kind="needle", num_history=512, needle_margin=0.0))


def test_needle_dominates_every_other_box():
    """workloads.py:80-85: the planted key's probe score beats every other
    physical page's box score by the margin."""
    spec = W.WorkloadSpec(kind="needle", num_history=2048, num_heads=2, head_dim=16, needle_margin=0.5, seed=4)
    w, t = W.gen_workload(spec)
    q, k = w.q[-1], w.k[:, 0]
    other = W.max_box_score(k, q, 64, {t.needle_pages[0]})
    assert (q @ k[t.needle_positions[0]]).max() >= other + 0.5 - 1e-9
