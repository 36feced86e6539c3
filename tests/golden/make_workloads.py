"""Golden fixture for the workload generator and the recall machinery
(tests/test_workloads.py, tests/test_gpu_recall.py), from the REAL reference.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_workloads.py

Imports ``sparsekv`` from /root/reference/pkg/src (read-only) and writes
workloads.json next to this script: sha256 digests of gen_workload's arrays
for a set of specs plus their ground truth, the reference's
sweeps.clustered_recall table and its C06 needle-recall numbers.  The
plotting module the sweeps import is stubbed (matplotlib is absent).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("SPARSEKV_REF", "/root/reference/pkg/src")
sys.dont_write_bytecode = True
sys.path.insert(0, REF)
for name in ("matplotlib", "matplotlib.pyplot"):  # report.py imports it at module level
    sys.modules.setdefault(name, types.ModuleType(name))
sys.modules["matplotlib"].use = lambda *a, **k: None
sys.modules["matplotlib"].pyplot = sys.modules["matplotlib.pyplot"]
sys.modules["matplotlib.pyplot"].rcParams = {}

from sparsekv import sweeps  # noqa: E402
from sparsekv.cache import HeadPages  # noqa: E402
from sparsekv.selector import exact_top_k_pages, select_pages  # noqa: E402
from sparsekv.workloads import WorkloadSpec, gen_workload  # noqa: E402

SPECS = [
    dict(kind="random", num_history=300, num_queries=5, num_heads=4, num_kv_heads=2, head_dim=16, seed=1),
    dict(kind="needle", num_history=512, head_dim=16, needle_margin=0.5, seed=7),
    dict(kind="needle", num_history=4096, num_heads=4, num_kv_heads=1, head_dim=64, needle_margin=1.0, seed=11),
    dict(kind="clustered_needles", num_history=2048, head_dim=16, needle_margin=0.75, cluster_span=2, seed=3),
    dict(kind="clustered_needles", num_history=1000, num_heads=8, num_kv_heads=2, head_dim=32,
         needle_margin=0.5, cluster_span=3, seed=5),
    dict(kind="needle", num_history=130, head_dim=16, seed=2),   # few pages: fallback free list
]


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, np.float64).tobytes()).hexdigest()


def needle_stats(trials, seed):
    """verify.py:219-248 with a configurable trial count."""
    hits = ohits = agree = 0
    for i in range(trials):
        spec = WorkloadSpec(kind="needle", num_history=512, num_queries=1, num_heads=1, num_kv_heads=1,
                            head_dim=16, needle_margin=0.5, physical_page=64, logical_page=16,
                            seed=seed * trials + i)
        w, truth = gen_workload(spec)
        head = HeadPages(0, 64, 16, bits=None, with_stats=True)
        head.append(w.k[:, 0, :], w.v[:, 0, :])
        q = w.q[-1, 0, :]
        sel = set(select_pages(q, head.live_pages(), 256, 64))
        orc = set(exact_top_k_pages(q, w.k[:, 0, :], 256, 64))
        h, o = truth.needle_pages[0] in sel, truth.needle_pages[0] in orc
        hits, ohits, agree = hits + h, ohits + o, agree + (h == o)
    return {"trials": trials, "recall": hits / trials, "oracle_recall": ohits / trials,
            "oracle_agreement": agree / trials}


def main():
    out = {"specs": []}
    for sp in SPECS:
        w, t = gen_workload(WorkloadSpec(**sp))
        out["specs"].append({"spec": sp, "q": digest(w.q), "k": digest(w.k), "v": digest(w.v),
                             "k_sum": float(np.asarray(w.k).sum()), "positions": list(t.needle_positions),
                             "pages": list(t.needle_pages)})
    budgets = (320, 384, 512, 768)
    table = sweeps.clustered_recall(budgets, trials=40, seed=0)
    out["clustered_recall"] = {"budgets": budgets, "trials": 40, "seed": 0,
                               "table": {str(b): table[b] for b in budgets}}
    out["needle_recall"] = needle_stats(400, 0)
    with open(os.path.join(HERE, "workloads.json"), "w") as fp:
        json.dump(out, fp, indent=1)
    print(json.dumps(out["clustered_recall"]), json.dumps(out["needle_recall"]))


if __name__ == "__main__":
    main()
