"""Run-to-run bitwise determinism (reference test_engine.py:260-279, C11):
two fresh engines on the same inputs give identical prefill outputs, decode
outputs, index tables and pages.  K4 work items, K2 scores/top-k and K3's
cluster merge all reduce in a fixed order (no float atomics)."""

import numpy as np
import pytest

import paper_2502_14866_b200 as sk
from test_gpu_edges import fp16_vals

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("bits", [4, None])
def test_engine_is_bitwise_deterministic(bits):
    rng = np.random.default_rng(31)
    n, h, h_kv, d = 1500, 16, 4, 128
    gates = rng.uniform(0, 1, h).tolist()
    q, k, v = fp16_vals(rng, n, h, d), fp16_vals(rng, n, h_kv, d), fp16_vals(rng, n, h_kv, d)
    steps = [(fp16_vals(rng, h, d), fp16_vals(rng, h_kv, d), fp16_vals(rng, h_kv, d)) for _ in range(6)]
    runs = []
    for _ in range(2):
        cfg = sk.EngineConfig(quant_bits=bits, budget_tokens=512, reuse_interval=3, local_blocks=2)
        eng = sk.Engine(cfg, sk.classify_heads(gates, 0.5, 1, 2), device="cuda:0")
        outs = [eng.prefill(sk.Workload(q, k, v))]
        tables = []
        for qn, kn, vn in steps:
            r = eng.decode_step(qn, kn, vn)
            outs.append(r.output)
            tables.append([tuple(t.positions) for t in r.index_tables])
        pages = [[(p.page_id, p.k_codes.tobytes(), p.v_codes.tobytes()) for p in eng.cache.pool_of(kv).live_pages()]
                 for kv in range(h_kv)]
        runs.append((outs, tables, pages))
    (o1, t1, p1), (o2, t2, p2) = runs
    for a, b in zip(o1, o2):
        np.testing.assert_array_equal(a, b)
    assert t1 == t2 and p1 == p2
