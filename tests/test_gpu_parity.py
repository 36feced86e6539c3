"""B200 parity: the CUDA path (through the C ABI) against the reference's
golden fixtures and the pinned CPU oracle.

Bit-exact: page statistics, codes, page bounds (scale/zero), selected page
indices, index tables, invoked flags, ledgers.  Tolerance (north_star):
attention outputs vs the reference's fp32 output, max-abs <= 2e-2 and
cosine >= 0.9999 per head.
"""

import os

import numpy as np
import pytest
import torch

import paper_2502_14866_b200 as sk
from oracle import sparsekv_oracle as O

pytestmark = pytest.mark.gpu

ATOL = 2e-2
MIN_COS = 0.9999


def load(golden_dir, name):
    return np.load(os.path.join(golden_dir, name))


def assert_close_attn(out, ref, atol=ATOL, min_cos=MIN_COS):
    out = np.asarray(out, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.abs(out - ref).max()
    assert err <= atol, f"max-abs {err:.3e} > {atol}"
    o = out.reshape(-1, out.shape[-1]) if out.ndim == 2 else out.transpose(1, 0, 2).reshape(out.shape[1], -1)
    r = ref.reshape(-1, ref.shape[-1]) if ref.ndim == 2 else ref.transpose(1, 0, 2).reshape(ref.shape[1], -1)
    cos = (o * r).sum(1) / (np.linalg.norm(o, axis=1) * np.linalg.norm(r, axis=1) + 1e-30)
    assert cos.min() >= min_cos, f"min cosine {cos.min():.7f} < {min_cos}"


def engine_from_golden(g):
    bits = int(g["quant_bits"]) or None
    cfg = sk.EngineConfig(quant_bits=bits, budget_tokens=int(g["budget"]), reuse_interval=int(g["reuse"]),
                          sink_blocks=int(g["sink"]), local_blocks=int(g["local"]),
                          target_sparsity=float(g["sparsity"]))
    prof = sk.classify_heads(g["gates"], cfg.target_sparsity, cfg.sink_blocks, cfg.local_blocks)
    return sk.Engine(cfg, prof, device="cuda:0"), bits


def check_snapshot(cache, g, prefix, bits):
    recs = []
    for dense, pool in ((1, cache.dense_pool), (0, cache.streaming_pool)):
        for kv in sorted(pool):
            for pg in pool[kv].live_pages():
                recs.append((dense, kv, pg))
    assert [r[0] for r in recs] == g[prefix + "page_dense"].tolist()
    assert [r[1] for r in recs] == g[prefix + "page_kv"].tolist()
    assert [r[2].page_id for r in recs] == g[prefix + "page_index"].tolist()
    assert [r[2].token_count for r in recs] == g[prefix + "page_tokens"].tolist()
    for i, (dense, kv, pg) in enumerate(recs):
        t = pg.token_count
        if bits:
            np.testing.assert_array_equal(pg.k_codes[:t], g[prefix + "k_codes"][i, :t])
            np.testing.assert_array_equal(pg.v_codes[:t], g[prefix + "v_codes"][i, :t])
        else:
            np.testing.assert_array_equal(pg.k_codes[:t], g[prefix + "k_codes"][i, :t].astype(np.float64))
            np.testing.assert_array_equal(pg.v_codes[:t], g[prefix + "v_codes"][i, :t].astype(np.float64))
        for name in ("k_scale", "k_zero", "v_scale", "v_zero"):
            np.testing.assert_array_equal(getattr(pg, name), g[prefix + name][i], err_msg=name)
        assert len(pg.stats) == (-(-t // 16) if dense else 0)
        for j, st in enumerate(pg.stats):
            np.testing.assert_array_equal(st.k_min, g[prefix + "stats_min"][i, j].astype(np.float64))
            np.testing.assert_array_equal(st.k_max, g[prefix + "stats_max"][i, j].astype(np.float64))
            assert st.covered_tokens == g[prefix + "stats_covered"][i, j]


@pytest.mark.parametrize("name", ["engine_kv4.npz", "engine_fp16pages.npz"])
def test_load_context_pages_bit_exact(golden_dir, name):
    g = load(golden_dir, name)
    eng, bits = engine_from_golden(g)
    eng.load_context(g["k"].astype(np.float32), g["v"].astype(np.float32))
    check_snapshot(eng.cache, g, "load_", bits)


@pytest.mark.parametrize("name", ["engine_kv4.npz", "engine_fp16pages.npz"])
def test_engine_prefill_and_decode_match_reference(golden_dir, name):
    g = load(golden_dir, name)
    eng, bits = engine_from_golden(g)
    f32 = lambda a: a.astype(np.float32)  # noqa: E731
    out = eng.prefill(sk.Workload(f32(g["q"]), f32(g["k"]), f32(g["v"])))
    assert_close_attn(out, g["prefill_out"])
    h = g["q"].shape[1]
    assert [eng.ledger.tiles[(sk.PREFILL, hh)] for hh in range(h)] == g["prefill_ledger"].tolist()
    check_snapshot(eng.cache, g, "load_", bits)
    for t in range(g["q_new"].shape[0]):
        res = eng.decode_step(f32(g["q_new"][t]), f32(g["k_new"][t]), f32(g["v_new"][t]))
        ref_tabs = [tuple(int(x) for x in row if x >= 0) for row in g["decode_tables"][t]]
        assert [tuple(tb.positions) for tb in res.index_tables] == ref_tabs, f"step {t}"
        assert [int(res.invoked.get(kv, -1)) for kv in range(g["k"].shape[1])] == g["decode_invoked"][t].tolist()
        assert_close_attn(res.output, g["decode_out"][t])
    assert [eng.ledger.tiles[(sk.DECODE, hh)] for hh in range(h)] == g["decode_ledger"].tolist()
    assert [eng.ledger.selector_invocations.get(kv, 0) for kv in range(g["k"].shape[1])] == \
        g["selector_calls"].tolist()
    check_snapshot(eng.cache, g, "final_", bits)


def test_select_pages_bit_exact(golden_dir):
    g = load(golden_dir, "select.npz")
    for i in range(int(g["n_cases"])):
        keys = g[f"c{i}_keys"].astype(np.float32)
        head = sk.HeadPages(0, 64, 16, bits=None, with_stats=True)
        head.append(keys, np.zeros_like(keys))
        pages = head.live_pages()
        q = g[f"c{i}_q"].astype(np.float64)
        assert sk.select_pages(q, pages, int(g[f"c{i}_budget"]), 64) == g[f"c{i}_sel"].tolist(), f"case {i}"
        np.testing.assert_array_equal(sk.score_pages(q, pages), g[f"c{i}_scores"])
    keys = np.zeros((64 * 40, 128), np.float32)
    head = sk.HeadPages(0, 64, 16, bits=None, with_stats=True)
    head.append(keys, keys)
    assert sk.select_pages(np.ones(128), head.live_pages(), 640, 64) == g["tie_sel"].tolist()


def test_quantize_page_bit_exact(golden_dir):
    g = load(golden_dir, "quantize.npz")
    for i in range(int(g["n_cases"])):
        codes, scale, zero = sk.quantize_page(g[f"q{i}_raw"].astype(np.float32), int(g[f"q{i}_bits"]))
        np.testing.assert_array_equal(codes, g[f"q{i}_codes"], err_msg=f"case {i}")
        np.testing.assert_array_equal(scale, g[f"q{i}_scale"], err_msg=f"case {i}")
        np.testing.assert_array_equal(zero, g[f"q{i}_zero"], err_msg=f"case {i}")


def test_blockwise_attention_matches_reference(golden_dir):
    g = load(golden_dir, "blockwise.npz")
    for i in range(int(g["n_cases"])):
        n, s, h, h_kv, tq, tk = g[f"b{i}_geom"].tolist()
        mask = g[f"b{i}_mask"]
        sched = {(hh, qt): np.nonzero(mask[hh, qt])[0].tolist() for hh in range(h) for qt in range(mask.shape[1])}
        f32 = lambda a: a.astype(np.float32)  # noqa: E731
        out, led = sk.blockwise_attention(sk.Workload(f32(g[f"b{i}_q"]), f32(g[f"b{i}_k"]), f32(g[f"b{i}_v"])),
                                          sched, tq, tk, "prefill")
        assert_close_attn(out, g[f"b{i}_out"])
        assert [led.tiles[("prefill", hh)] for hh in range(h)] == g[f"b{i}_ledger"].tolist()


def test_prefill_8k_against_oracle_sampled_tiles():
    """cfg1 geometry (32/8/128, 50% streaming, sink 1 + local 4): full GPU
    prefill, oracle on sampled query tiles (slicing is exact)."""
    rng = np.random.default_rng(11)
    n = s = 8192
    h, h_kv, d = 32, 8, 128
    gates = [0.9 - 0.001 * i if i % 4 < 2 else 0.1 + 0.001 * i for i in range(h)]
    cfg = sk.EngineConfig(quant_bits=4, local_blocks=4)
    prof = sk.classify_heads(gates, 0.5, 1, 4)
    q = torch.randn(n, h, d, device="cuda", dtype=torch.float16)
    k = torch.randn(s, h_kv, d, device="cuda", dtype=torch.float16)
    v = torch.randn(s, h_kv, d, device="cuda", dtype=torch.float16)
    eng = sk.Engine(cfg, prof, device="cuda:0")
    out = eng.prefill(sk.Workload(q, k, v)).float().cpu().numpy()
    roles = O.assign_roles(gates, 0.5, 1, 4)
    qh, kh, vh = (t.float().cpu().numpy() for t in (q, k, v))
    for qt in (0, 1, 5, 63, 64, 127):
        r0, r1 = qt * 64, qt * 64 + 64
        sched = {}
        n_tiles = s // 64
        for hh in range(h):
            dg = qt
            sched[(hh, 0)] = list(range(dg + 1)) if roles[hh].role == O.RETRIEVAL else \
                O.lambda_tiles(n_tiles, 1, 4, dg)
        ref, _ = O.tiled_attention(qh[r0:r1], kh[:r1], vh[:r1], sched, 64, 64)
        assert_close_attn(out[r0:r1], ref)
    led = eng.ledger
    n_qt = n // 64
    exp_vis = sum(qt + 1 if roles[hh].role == O.RETRIEVAL else len(O.lambda_tiles(n_qt, 1, 4, qt))
                  for hh in range(h) for qt in range(n_qt))
    assert led.visited(sk.PREFILL) == exp_vis == 142_176  # cfg1 visited tiles
    assert led.total(sk.PREFILL) == 264_192


def test_prefill_256k_against_oracle_sampled_tiles():
    """cfg3 geometry for one layer (32/8/128 at 256k, balanced heads): the
    device prefill's sampled query tiles -- first, middle, last -- against the
    oracle on the same inputs, and the visited-tile ledger."""
    n = s = 262144
    h, h_kv, d = 32, 8, 128
    gates = [0.9 - 0.001 * i if i % 4 < 2 else 0.1 + 0.001 * i for i in range(h)]
    cfg = sk.EngineConfig(quant_bits=4, local_blocks=4)
    prof = sk.classify_heads(gates, 0.5, 1, 4)
    g = torch.Generator(device="cuda").manual_seed(256)
    q = torch.randn(n, h, d, device="cuda", dtype=torch.float16, generator=g)
    k = torch.randn(s, h_kv, d, device="cuda", dtype=torch.float16, generator=g)
    v = torch.randn(s, h_kv, d, device="cuda", dtype=torch.float16, generator=g)
    eng = sk.Engine(cfg, prof, device="cuda:0", capacity_tokens=s)
    out = eng.prefill_device(q, k, v, d)
    roles = O.assign_roles(gates, 0.5, 1, 4)
    n_tiles = s // 64
    for qt in (0, 2049, n_tiles - 1):
        r0, r1 = qt * 64, qt * 64 + 64
        sched = {(hh, 0): list(range(qt + 1)) if roles[hh].role == O.RETRIEVAL else O.lambda_tiles(n_tiles, 1, 4, qt)
                 for hh in range(h)}
        qh, kh, vh = (t.float().cpu().numpy() for t in (q[r0:r1], k[:r1], v[:r1]))
        ref, _ = O.tiled_attention(qh, kh, vh, sched, 64, 64)
        assert_close_attn(out[r0:r1].float().cpu().numpy(), ref)
    exp_vis = sum(qt + 1 if roles[hh].role == O.RETRIEVAL else len(O.lambda_tiles(n_tiles, 1, 4, qt))
                  for hh in range(h) for qt in range(n_tiles))
    assert eng.ledger.visited(sk.PREFILL) == exp_vis == 134_578_016  # DESIGN 9: cfg3 visited tiles


def test_decode_long_context_selection_matches_oracle():
    """16k-token context, budget 1024, reuse 4: 12 decode steps; selections,
    index tables and outputs against the oracle driven on the same data."""
    rng = np.random.default_rng(12)
    s, h, h_kv, d = 16384, 8, 2, 128
    gates = [0.9, 0.8, 0.1, 0.2, 0.85, 0.15, 0.12, 0.11]
    cfg = sk.EngineConfig(quant_bits=4, budget_tokens=1024, reuse_interval=4, local_blocks=4)
    prof = sk.classify_heads(gates, 0.5, 1, 4)
    k = rng.standard_normal((s, h_kv, d)).astype(np.float16).astype(np.float32)
    v = rng.standard_normal((s, h_kv, d)).astype(np.float16).astype(np.float32)
    eng = sk.Engine(cfg, prof, device="cuda:0")
    eng.load_context(k, v)
    ref = O.OracleEngine(O.Config(quant_bits=4, budget_tokens=1024, reuse_interval=4, local_blocks=4),
                         O.assign_roles(gates, 0.5, 1, 4))
    ref.load_context(k, v)
    for t in range(12):
        qn = rng.standard_normal((h, d)).astype(np.float16).astype(np.float32)
        kn = rng.standard_normal((h_kv, d)).astype(np.float16).astype(np.float32)
        vn = rng.standard_normal((h_kv, d)).astype(np.float16).astype(np.float32)
        res = eng.decode_step(qn, kn, vn)
        rr = ref.decode_step(qn, kn, vn)
        assert [tuple(tb.positions) for tb in res.index_tables] == rr.tables, f"step {t}"
        assert res.invoked == rr.invoked
        assert_close_attn(res.output, rr.output)
    assert eng.ledger.tiles == {k2: v2 for k2, v2 in ref.tally.tiles.items()}


def test_decode_graph_matches_eager_engine():
    """The CUDA-graph multi-layer decode runner reproduces Engine.decode_step
    (same selections -> same outputs, same ledger) for 2 layers x 9 steps."""
    from paper_2502_14866_b200.decode_graph import DecodeGraph

    rng = np.random.default_rng(13)
    s, h, h_kv, d, L = 4096 + 37, 8, 2, 128, 2
    gates = [0.9, 0.8, 0.1, 0.2, 0.85, 0.15, 0.12, 0.11]
    cfg = sk.EngineConfig(quant_bits=4, budget_tokens=512, reuse_interval=4, local_blocks=4)
    prof = sk.classify_heads(gates, 0.5, 1, 4)
    ks = [rng.standard_normal((s, h_kv, d)).astype(np.float16) for _ in range(L)]
    vs = [rng.standard_normal((s, h_kv, d)).astype(np.float16) for _ in range(L)]
    eager = [sk.Engine(cfg, prof, device="cuda:0") for _ in range(L)]
    graph = [sk.Engine(cfg, prof, device="cuda:0") for _ in range(L)]
    for e1, e2, k, v in zip(eager, graph, ks, vs):
        e1.load_context(k.astype(np.float32), v.astype(np.float32))
        e2.load_context(k.astype(np.float32), v.astype(np.float32))
    dg = DecodeGraph(graph, 16, d)
    for t in range(9):
        qn = torch.from_numpy(rng.standard_normal((L, h, d)).astype(np.float16)).cuda()
        kn = torch.from_numpy(rng.standard_normal((L, h_kv, d)).astype(np.float16)).cuda()
        vn = torch.from_numpy(rng.standard_normal((L, h_kv, d)).astype(np.float16)).cuda()
        dg.q.copy_(qn)
        dg.k.copy_(kn)
        dg.v.copy_(vn)
        out_g = dg.step().float().cpu().numpy()
        for li in range(L):
            res = eager[li].decode_step(qn[li], kn[li], vn[li])
            np.testing.assert_allclose(out_g[li], res.output.float().cpu().numpy(), atol=1e-3, rtol=0)
    for e1, e2 in zip(eager, graph):
        assert e1.ledger.tiles == e2.ledger.tiles
        assert e1.ledger.selector_invocations == e2.ledger.selector_invocations


def _oracle_pages(ref_pools):
    out = []
    for dense, pool in ((1, ref_pools.dense), (0, ref_pools.streaming)):
        for kv in sorted(pool):
            for pg in pool[kv].live():
                out.append((dense, kv, pg))
    return out


@pytest.mark.parametrize("bits", [4, 8, 3, None])
def test_decode_appends_bit_exact_across_formats(bits):
    """Misaligned context (1000 tokens, open page of 40) + 40 decode steps:
    every page (codes, scale/zero, logical stats) equals the oracle's after
    the fused incremental / page-opening appends; outputs within tolerance."""
    rng = np.random.default_rng(21 + (bits or 0))
    s, h, h_kv, d = 1000, 8, 2, 128
    gates = [0.9, 0.1, 0.8, 0.2, 0.05, 0.15, 0.12, 0.11]  # kv 1 all-streaming -> ring pool
    cfg = sk.EngineConfig(quant_bits=bits, budget_tokens=384, reuse_interval=3, local_blocks=2)
    prof = sk.classify_heads(gates, 0.75, 1, 2)
    k = rng.standard_normal((s, h_kv, d)).astype(np.float16).astype(np.float32)
    v = rng.standard_normal((s, h_kv, d)).astype(np.float16).astype(np.float32)
    eng = sk.Engine(cfg, prof, device="cuda:0")
    eng.load_context(k, v)
    ref = O.OracleEngine(O.Config(quant_bits=bits, budget_tokens=384, reuse_interval=3, local_blocks=2),
                         O.assign_roles(gates, 0.75, 1, 2))
    ref.load_context(k, v)
    for t in range(40):
        scale = 1.0 + 3.0 * (t % 5 == 0)  # occasional out-of-range tokens move page bounds
        qn = rng.standard_normal((h, d)).astype(np.float16).astype(np.float32)
        kn = (rng.standard_normal((h_kv, d)) * scale).astype(np.float16).astype(np.float32)
        vn = (rng.standard_normal((h_kv, d)) * scale).astype(np.float16).astype(np.float32)
        res = eng.decode_step(qn, kn, vn)
        rr = ref.decode_step(qn, kn, vn)
        assert [tuple(tb.positions) for tb in res.index_tables] == rr.tables, f"step {t}"
        assert_close_attn(res.output, rr.output)
    mine = [(1, kv, pg) for kv in sorted(eng.cache.dense_pool) for pg in eng.cache.dense_pool[kv].live_pages()] + \
           [(0, kv, pg) for kv in sorted(eng.cache.streaming_pool) for pg in eng.cache.streaming_pool[kv].live_pages()]
    theirs = _oracle_pages(ref.pools)
    assert [(a, b, c.page_id, c.token_count) for a, b, c in mine] == \
        [(a, b, c.index, c.tokens) for a, b, c in theirs]
    for (_, _, pg), (_, _, rp) in zip(mine, theirs):
        t = pg.token_count
        np.testing.assert_array_equal(pg.k_codes[:t], rp.k_codes[:t])
        np.testing.assert_array_equal(pg.v_codes[:t], rp.v_codes[:t])
        for name in ("k_scale", "k_zero", "v_scale", "v_zero"):
            np.testing.assert_array_equal(getattr(pg, name), getattr(rp, name))
        assert len(pg.stats) == len(rp.bounds)
        for st, (kmin, kmax, cov) in zip(pg.stats, rp.bounds):
            np.testing.assert_array_equal(st.k_min, kmin)
            np.testing.assert_array_equal(st.k_max, kmax)
            assert st.covered_tokens == cov


def _tie_grid(rng, shape):
    """Values on a 1/8 grid in [-2, 2] with both ends present per channel:
    (x - lo) / scale hits exact .5 ties (x = 0 -> 7.5 for 4-bit codes)."""
    x = rng.integers(-16, 17, shape).astype(np.float32) / 8.0
    x[0], x[1] = -2.0, 2.0
    return x


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16], ids=["f16", "bf16"])
@pytest.mark.parametrize("dist", ["normal", "wide", "ties"])
@pytest.mark.parametrize("bits", [4, 2])
def test_bulk_append_pages_bit_exact(dtype, dist, bits):
    """K1's full-page fast path (KV<=4, D 128, page 64) and the generic
    rebuild, through load_context (page-aligned start) and a chunk appended
    at an unaligned start: every page's codes, scale/zero and logical stats
    equal the oracle's -- including exact .5 ties (round half to even) and
    wide-range values."""
    rng = np.random.default_rng(hash((str(dtype), dist, bits)) % 2**32)
    s, n2, h, h_kv, d = 1000, 300, 8, 2, 128

    def vals(*shape):
        if dist == "normal":
            x = rng.standard_normal(shape).astype(np.float32)
        elif dist == "wide":
            x = (rng.choice([-1, 1], shape) * np.exp2(rng.uniform(-12, 12, shape))).astype(np.float32)
        else:
            x = _tie_grid(rng, shape)
        return torch.from_numpy(x).to(dtype).float().numpy()

    gates = [0.9, 0.1, 0.8, 0.2, 0.05, 0.15, 0.12, 0.11]  # kv 1 all-streaming -> ring pool
    kw = dict(quant_bits=bits, budget_tokens=384, reuse_interval=3, local_blocks=2)
    prof = sk.classify_heads(gates, 0.75, 1, 2)
    k, v = vals(s, h_kv, d), vals(s, h_kv, d)
    eng = sk.Engine(sk.EngineConfig(**kw), prof, device="cuda:0", dtype=dtype)
    eng.load_context(torch.from_numpy(k).to(dtype).cuda(), torch.from_numpy(v).to(dtype).cuda())
    ref = O.OracleEngine(O.Config(**kw), O.assign_roles(gates, 0.75, 1, 2))
    ref.load_context(k, v)
    q2 = torch.from_numpy(rng.standard_normal((n2, h, d)).astype(np.float32)).to(dtype).float().numpy()
    k2, v2 = vals(n2, h_kv, d), vals(n2, h_kv, d)
    eng.prefill_chunk(sk.Workload(*(torch.from_numpy(a).to(dtype).cuda() for a in (q2, k2, v2))))
    ref.prefill_chunk(q2, k2, v2)
    mine = [(1, kv, pg) for kv in sorted(eng.cache.dense_pool) for pg in eng.cache.dense_pool[kv].live_pages()] + \
           [(0, kv, pg) for kv in sorted(eng.cache.streaming_pool) for pg in eng.cache.streaming_pool[kv].live_pages()]
    theirs = _oracle_pages(ref.pools)
    assert [(a, b, c.page_id, c.token_count) for a, b, c in mine] == \
        [(a, b, c.index, c.tokens) for a, b, c in theirs]
    for (_, _, pg), (_, _, rp) in zip(mine, theirs):
        t = pg.token_count
        np.testing.assert_array_equal(pg.k_codes[:t], rp.k_codes[:t])
        np.testing.assert_array_equal(pg.v_codes[:t], rp.v_codes[:t])
        for name in ("k_scale", "k_zero", "v_scale", "v_zero"):
            np.testing.assert_array_equal(getattr(pg, name), getattr(rp, name))
        for st, (kmin, kmax, cov) in zip(pg.stats, rp.bounds):
            np.testing.assert_array_equal(st.k_min, kmin)
            np.testing.assert_array_equal(st.k_max, kmax)
            assert st.covered_tokens == cov
