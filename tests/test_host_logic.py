"""Host-side integer logic of the package against the oracle and the
reference's known answers (CPU only): head classification, Lambda
schedules, pins, reuse rule, ledger / cost report, config validation.  These
decide block masks, index tables and ledgers, which must match bit-exactly
(SURVEY 8(c))."""

import json

import numpy as np
import pytest

import paper_2502_14866_b200 as sk
from oracle import sparsekv_oracle as O
from paper_2502_14866_b200.heads import lambda_segments
from paper_2502_14866_b200.selector import selection_size


def test_classify_heads_known_answers_and_oracle():
    prof = sk.classify_heads([0.1, 0.9, 0.4, 0.8], 0.5, 1, 2)  # test_heads.py:23-27
    assert [p.head for p in prof if p.role == sk.RETRIEVAL] == [1, 3]
    rng = np.random.default_rng(0)
    for trial in range(50):
        h = int(rng.integers(1, 40))
        gates = rng.uniform(0, 1, h).round(int(rng.integers(1, 3))).tolist()  # rounding forces ties
        sp = float(rng.choice([0.0, 0.25, 0.5, 0.75, 0.9]))
        ours = [p.role for p in sk.classify_heads(gates, sp, 1, 4)]
        ref = [r.role for r in O.assign_roles(gates, sp, 1, 4)]
        assert ours == ref, (trial, gates, sp)


def test_streaming_schedule_matches_oracle():
    assert sk.streaming_schedule(2000, sk.HeadProfile(0, 0.1, sk.STREAMING, 1, 2), 1999).tiles() == [0, 1998, 1999]
    for n in (1, 2, 3, 7, 64, 2048):
        for sink in (1, 2):
            for local in (1, 2, 4):
                for qt in range(0, n, max(1, n // 17)):
                    segs = lambda_segments(n, sink, local, qt)
                    tiles = [t for a, b in segs for t in range(a, b)]
                    assert tiles == O.lambda_tiles(n, sink, local, qt), (n, sink, local, qt)
                    assert len(segs) <= 2


def test_pins_and_selection_size():
    assert sk.selector.pinned_pages(8) == [0, 6, 7]        # test_selector.py:120-128
    assert sk.selector.pinned_pages(2) == [0, 1]
    assert sk.selector.pinned_pages(1) == [0]
    for n in range(1, 200):
        for k in (1, 2, 3, 4, 64):
            expect = n if k >= n else (len(O.pins(n)) if k <= len(O.pins(n)) else k)
            assert selection_size(n, k) == expect, (n, k)


def test_reuse_rule_invocation_counts():
    """ceil(T / C) selector invocations over T consecutive steps
    (test_selector.py:178-191), through SelectionState.valid_for."""
    for c in (1, 2, 3, 4, 7):
        for steps in (1, 5, 16, 33):
            st, calls = None, 0
            for step in range(steps):
                if not (st is not None and st.valid_for(step, 4096, c)):
                    st = sk.SelectionState([0], step, c, 4096)
                    calls += 1
            assert calls == -(-steps // c)
    st = sk.SelectionState([0], 0, 4, 4096)
    assert not st.valid_for(1, 2048, 4)  # budget change invalidates (selector.py:120-125)
    assert not st.valid_for(1, 4096, 2)  # interval change invalidates


def test_ledger_and_cost_report():
    led = sk.CostLedger()
    led.record_tiles("prefill", 0, 10, 21)            # the 10-of-21 -> 2.1x example
    led.record_selector(3)
    led.record_selector(3)
    rep = sk.cost_report(led)
    assert rep["stages"]["prefill"]["speedup"] == pytest.approx(2.1)
    assert rep["stages"]["prefill"]["visited_tiles"] == 10 and rep["stages"]["prefill"]["total_tiles"] == 21
    assert rep["selector_invocations"]["total"] == 2
    assert rep["selector_invocations"]["per_kv_head"] == {"3": 2}
    with pytest.raises(ValueError):
        led.record_tiles("prefill", 0, 5, 4)           # visited > total (ledger.py:15-36)


def test_engine_config_validation_and_json(tmp_path):
    cfg = sk.EngineConfig(quant_bits=0)
    assert cfg.quant_bits is None                      # 0 -> None (engine.py:43-67)
    for bad, msg in ((dict(physical_page=48, logical_page=32), "divide"), (dict(quant_bits=9), "quant_bits"),
                     (dict(budget_tokens=16), "budget")):
        with pytest.raises(ValueError, match=msg):
            sk.EngineConfig(**bad)
    p = tmp_path / "cfg.json"
    p.write_text(json.dumps({"budget_tokens": 2048, "reuse_interval": 2}))
    cfg = sk.EngineConfig.from_json(p)
    assert (cfg.budget_tokens, cfg.reuse_interval) == (2048, 2)
    p.write_text(json.dumps({"budget_tokens": 2048, "nope": 1}))
    with pytest.raises(ValueError, match="unknown config keys"):
        sk.EngineConfig.from_json(p)


def test_block_iterator_semantics():
    it = sk.BlockIterator(((0, 1), (9, 11)))
    assert it.tiles() == [0, 9, 10] and len(it) == 3     # test_heads.py:73-76
    with pytest.raises(ValueError):
        sk.BlockIterator(((5, 7), (6, 9)))
    with pytest.raises(ValueError):
        sk.BlockIterator(((3, 3),))


def test_load_gates_reads_per_layer_arrays(tmp_path):
    """heads.py:128-136: one layer of a JSON array of per-layer gate arrays."""
    import json

    import paper_2502_14866_b200 as sk
    path = tmp_path / "gates.json"
    path.write_text(json.dumps([[0.9, 0.1, 0.3], [0.5, 0.4, 1], [0, 0.25, 0.75]]))
    assert sk.load_gates(path) == [0.9, 0.1, 0.3]
    assert sk.load_gates(str(path), 1) == [0.5, 0.4, 1.0]
    assert all(isinstance(g, float) for g in sk.load_gates(path, 2))
    with pytest.raises(ValueError, match="outside"):
        sk.load_gates(path, 3)
    with pytest.raises(ValueError, match="outside"):
        sk.load_gates(path, -1)
    bad = tmp_path / "bad.json"
    for doc in ([], {"layers": []}):
        bad.write_text(json.dumps(doc))
        with pytest.raises(ValueError, match="non-empty JSON array"):
            sk.load_gates(bad)
    # the profiles of a loaded layer, like the reference's per-layer oracle
    prof = sk.classify_heads(sk.load_gates(path, 2), 0.5, 1, 4)
    assert [p.role for p in prof] == [sk.STREAMING, sk.RETRIEVAL, sk.RETRIEVAL]


def test_page_table_standalone_api():
    """cache.py:109-140: PageTable(page_size) with register / evict / lookup."""
    import paper_2502_14866_b200 as sk
    t = sk.PageTable(64)
    t.register(0, 10)
    t.register(2, 12)
    t.register(1, 11)
    t.num_tokens = 150
    assert t.live_indices == [0, 1, 2] and t.page_ids == [10, 11, 12]
    assert t.lookup(0) == (10, 0) and t.lookup(130) == (12, 2)
    t.evict(1)
    with pytest.raises(KeyError, match="evicted"):
        t.lookup(64)
    with pytest.raises(IndexError, match="outside"):
        t.lookup(150)
    assert t.page_ids == [10, 12]
