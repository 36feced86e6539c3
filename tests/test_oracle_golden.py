"""Pin the CPU oracle to the real reference: every golden fixture in
tests/golden (made by tests/golden/make_golden.py from /root/reference) must
be reproduced -- bit-exactly for schedules, ledgers, selections, codes and
page statistics; to 1e-12 relative for float outputs."""

import os

import numpy as np
import pytest

from oracle import sparsekv_oracle as O


def load(golden_dir, name):
    return np.load(os.path.join(golden_dir, name))


def rel_err(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)


def check_snapshot(pools, g, prefix, bits):
    recs = []
    for dense, pool in ((1, pools.dense), (0, pools.streaming)):
        for kv in sorted(pool):
            for pg in pool[kv].live():
                recs.append((dense, kv, pg))
    assert [r[0] for r in recs] == g[prefix + "page_dense"].tolist()
    assert [r[1] for r in recs] == g[prefix + "page_kv"].tolist()
    assert [r[2].index for r in recs] == g[prefix + "page_index"].tolist()
    assert [r[2].tokens for r in recs] == g[prefix + "page_tokens"].tolist()
    for i, (dense, kv, pg) in enumerate(recs):
        t = pg.tokens
        if bits:
            np.testing.assert_array_equal(pg.k_codes[:t], g[prefix + "k_codes"][i, :t])
            np.testing.assert_array_equal(pg.v_codes[:t], g[prefix + "v_codes"][i, :t])
        else:
            np.testing.assert_array_equal(pg.k_codes[:t], g[prefix + "k_codes"][i, :t].astype(np.float64))
        for name in ("k_scale", "k_zero", "v_scale", "v_zero"):
            np.testing.assert_array_equal(getattr(pg, name), g[prefix + name][i])
        for j, (kmin, kmax, cov) in enumerate(pg.bounds):
            np.testing.assert_array_equal(kmin, g[prefix + "stats_min"][i, j].astype(np.float64))
            np.testing.assert_array_equal(kmax, g[prefix + "stats_max"][i, j].astype(np.float64))
            assert cov == g[prefix + "stats_covered"][i, j]
        if not dense:
            assert pg.bounds == []


@pytest.mark.parametrize("name", ["engine_kv4.npz", "engine_fp16pages.npz"])
def test_oracle_engine_matches_reference(golden_dir, name):
    g = load(golden_dir, name)
    bits = int(g["quant_bits"]) or None
    cfg = O.Config(quant_bits=bits, budget_tokens=int(g["budget"]), reuse_interval=int(g["reuse"]),
                   sink_blocks=int(g["sink"]), local_blocks=int(g["local"]),
                   target_sparsity=float(g["sparsity"]))
    roles = O.assign_roles(g["gates"], cfg.target_sparsity, cfg.sink_blocks, cfg.local_blocks)
    assert [r.role == O.RETRIEVAL for r in roles] == g["roles"].astype(bool).tolist()
    eng = O.OracleEngine(cfg, roles)
    f32 = lambda a: a.astype(np.float32)  # noqa: E731
    out = eng.prefill(f32(g["q"]), f32(g["k"]), f32(g["v"]))
    assert rel_err(out, g["prefill_out"]) <= 1e-6
    h = g["q"].shape[1]
    assert [eng.tally.tiles[(O.PREFILL, hh)] for hh in range(h)] == g["prefill_ledger"].tolist()
    for t in range(g["q_new"].shape[0]):
        st = eng.decode_step(f32(g["q_new"][t]), f32(g["k_new"][t]), f32(g["v_new"][t]))
        assert rel_err(st.output, g["decode_out"][t]) <= 1e-6
        ref_tabs = [tuple(int(x) for x in row if x >= 0) for row in g["decode_tables"][t]]
        assert st.tables == ref_tabs
        assert [int(st.invoked.get(kv, -1)) for kv in range(g["k"].shape[1])] == g["decode_invoked"][t].tolist()
    assert [eng.tally.tiles[(O.DECODE, hh)] for hh in range(h)] == g["decode_ledger"].tolist()
    assert [eng.tally.selector.get(kv, 0) for kv in range(g["k"].shape[1])] == g["selector_calls"].tolist()
    check_snapshot(eng.pools, g, "final_", bits)
    eng2 = O.OracleEngine(cfg, roles)
    eng2.load_context(f32(g["k"]), f32(g["v"]))
    check_snapshot(eng2.pools, g, "load_", bits)


def test_oracle_selector_matches_reference(golden_dir):
    g = load(golden_dir, "select.npz")
    for i in range(int(g["n_cases"])):
        keys = g[f"c{i}_keys"].astype(np.float64)
        head = O.PagedHead(64, 16, None, True)
        head.append(keys, np.zeros_like(keys))
        q = g[f"c{i}_q"].astype(np.float64)
        sc = O.eq2_scores(q, head.live())
        np.testing.assert_array_equal(sc, g[f"c{i}_scores"])  # exact: fp16-valued inputs
        sel = O.top_pages(q, head.live(), int(g[f"c{i}_budget"]), 64)
        assert sel == g[f"c{i}_sel"].tolist()
    keys = np.zeros((64 * 40, 128))
    head = O.PagedHead(64, 16, None, True)
    head.append(keys, keys)
    assert O.top_pages(np.ones(128), head.live(), 640, 64) == g["tie_sel"].tolist()


def test_oracle_sequential_eq2_equals_reference_blas(golden_dir):
    """Appendix A.4: on fp16-valued inputs a sequential fp64 Eq. 2 loop
    (the GPU's arithmetic order) reproduces the reference's BLAS scores."""
    g = load(golden_dir, "select.npz")
    for i in range(int(g["n_cases"])):
        keys = g[f"c{i}_keys"].astype(np.float64)
        q = g[f"c{i}_q"].astype(np.float64)
        n_log = -(-keys.shape[0] // 16)
        seq = np.full(-(-keys.shape[0] // 64), -np.inf)
        for lp in range(n_log):
            blk = keys[lp * 16:(lp + 1) * 16]
            kmin, kmax = blk.min(axis=0), blk.max(axis=0)
            for r in range(q.shape[0]):
                acc = 0.0
                for c in range(128):
                    acc += max(q[r, c] * kmax[c], q[r, c] * kmin[c])
                seq[lp // 4] = max(seq[lp // 4], acc)
        np.testing.assert_array_equal(seq, g[f"c{i}_scores"])


def test_oracle_quantize_matches_reference(golden_dir):
    g = load(golden_dir, "quantize.npz")
    for i in range(int(g["n_cases"])):
        codes, scale, zero = O.quantize(g[f"q{i}_raw"].astype(np.float64), int(g[f"q{i}_bits"]))
        np.testing.assert_array_equal(codes, g[f"q{i}_codes"])
        np.testing.assert_array_equal(scale, g[f"q{i}_scale"])
        np.testing.assert_array_equal(zero, g[f"q{i}_zero"])


def test_oracle_blockwise_matches_reference(golden_dir):
    g = load(golden_dir, "blockwise.npz")
    for i in range(int(g["n_cases"])):
        n, s, h, h_kv, tq, tk = g[f"b{i}_geom"].tolist()
        mask = g[f"b{i}_mask"]
        sched = {(hh, qt): np.nonzero(mask[hh, qt])[0].tolist()
                 for hh in range(h) for qt in range(mask.shape[1])}
        f32 = lambda a: a.astype(np.float32)  # noqa: E731
        out, tally = O.tiled_attention(f32(g[f"b{i}_q"]), f32(g[f"b{i}_k"]), f32(g[f"b{i}_v"]),
                                       sched, tq, tk, O.PREFILL)
        assert rel_err(out, g[f"b{i}_out"]) <= 1e-6
        assert [tally.tiles[(O.PREFILL, hh)] for hh in range(h)] == g[f"b{i}_ledger"].tolist()
        assert [O.diagonal(qt, tq, tk, n, s) for qt in range(mask.shape[1])] == g[f"b{i}_diag"].tolist()


# -- the reference's own known-answer tests, restated against the oracle ------


def test_known_answers_geometry_and_heads():
    assert O.kv_group(13, 4) == 3                                   # test_attn.py:66-68
    assert O.ceil_div(130, 64) == 3                                 # test_attn.py:349-353
    assert O.diagonal(1, 64, 64, 100, 132) == 2
    roles = O.assign_roles([0.1, 0.9, 0.4, 0.8], 0.5)               # test_heads.py:23-27
    assert [r.head for r in roles if r.role == O.RETRIEVAL] == [1, 3]
    assert O.lambda_tiles(2000, 1, 2, 1999) == [0, 1998, 1999]      # test_heads.py:103-105
    assert O.lambda_tiles(2, 1, 2, 1) == [0, 1]                     # test_heads.py:108-110
    for n_t in (10, 100, 1000):                                     # test_heads.py:125-131
        assert len(O.lambda_tiles(n_t, 1, 2, n_t - 1)) == 3


def test_known_answers_selector():
    assert O.pins(8) == [0, 6, 7] and O.pins(2) == [0, 1]           # test_selector.py:120-128
    q = np.array([1.0, -1.0])
    assert O.eq2_scalar(q, np.array([-1.0, -2.0]), np.array([2.0, 3.0])) == 4.0  # :32-42
    head = O.PagedHead(64, 16, None, True)                          # :138-145
    z = np.zeros((4 * 64, 2))
    head.append(z, z)
    assert O.top_pages(np.ones(2), head.live(), 64, 64) == [0, 2, 3]
    assert O.top_pages(np.ones(2), head.live(), 4 * 57, 64) == [0, 1, 2, 3]
    rng = np.random.default_rng(5)                                  # :111-117
    k = rng.standard_normal((128 * 64, 8))
    head = O.PagedHead(64, 16, None, True)
    head.append(k, k)
    assert len(O.top_pages(rng.standard_normal(8), head.live(), 4096, 64)) == 64


@pytest.mark.parametrize("interval,steps,expected", [(4, 16, 4), (2, 16, 8), (8, 16, 2), (16, 16, 1), (3, 10, 4)])
def test_known_answers_reuse(interval, steps, expected):                 # test_selector.py:178-191
    rng = np.random.default_rng(10)
    head = O.PagedHead(64, 16, None, True)
    k = rng.standard_normal((512, 8))
    head.append(k, k)
    q = rng.standard_normal(8)
    st, calls = None, 0
    for step in range(steps):
        _, st, ran = O.reuse_or_select(st, step, q, head.live(), 256, interval, 64)
        calls += ran
    assert calls == expected


def test_known_answers_streaming_pool_and_engine():
    rng = np.random.default_rng(9)                                  # test_cache.py:186-198
    head = O.PagedHead(64, 16, 4, False, (1, 2))
    for _ in range(50):
        b = rng.standard_normal((37, 4))
        head.append(b, b)
        assert len(head.live()) <= 4
    # exactly sink + local live pages (Appendix A.11)
    assert sorted(head.pages) == [0, head.page_count - 2, head.page_count - 1]
    rng = np.random.default_rng(5)                                  # test_engine.py:161-171
    eng = O.OracleEngine(O.Config(quant_bits=None), [O.Role(0, 0.1, O.STREAMING, 1, 2)])
    eng.load_context(rng.standard_normal((64 * 128, 1, 8)), rng.standard_normal((64 * 128, 1, 8)))
    st = eng.decode_step(rng.standard_normal((1, 8)), rng.standard_normal((1, 8)), rng.standard_normal((1, 8)))
    assert len(st.tables[0]) == 3 and eng.tally.tiles[(O.DECODE, 0)] == [3, 128]
    rng = np.random.default_rng(15)                                 # test_engine.py:174-203
    eng = O.OracleEngine(O.Config(quant_bits=None, budget_tokens=100_000),
                         [O.Role(0, 0.9, O.RETRIEVAL), O.Role(1, 0.1, O.STREAMING)])
    eng.load_context(rng.standard_normal((640, 1, 8)), rng.standard_normal((640, 1, 8)))
    st = eng.decode_step(rng.standard_normal((2, 8)), rng.standard_normal((1, 8)), rng.standard_normal((1, 8)))
    assert st.tables[1] == (0, 8, 9)


def test_exact_attention_matches_blockwise_full_schedule():
    rng = np.random.default_rng(0)                                  # test_attn.py:216-231
    q, k, v = (rng.standard_normal(s) for s in ((100, 2, 8), (160, 2, 8), (160, 2, 8)))
    sched = {(h, qt): O.dense_tiles(qt, 64, 64, 100, 160) for h in range(2) for qt in range(2)}
    out, _ = O.tiled_attention(q, k, v, sched, 64, 64)
    assert rel_err(out, O.exact_attention(q, k, v)) <= 1e-10
