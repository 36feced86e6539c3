"""B200 parity on the edge cases the reference's own tests exercise, against
the pinned CPU oracle: ragged and non-square prefill (S > N), MHA and wide
GQA groups, head_dim 64 and padded dims, bf16, all-streaming layers,
degenerate budgets (all pages / pins only), decoding at 128k context, and
KV-head shards recombining to the unsharded result."""

import numpy as np
import pytest
import torch

import paper_2502_14866_b200 as sk
from oracle import sparsekv_oracle as O
from paper_2502_14866_b200.sharding import shard_decode_inputs, shard_heads, shard_prefill_inputs, shard_profiles

pytestmark = pytest.mark.gpu

ATOL = 2e-2
MIN_COS = 0.9999


def close(out, ref, atol=ATOL):
    out = np.asarray(out, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.abs(out - ref).max()
    assert err <= atol, f"max-abs {err:.3e}"
    o = out.reshape(-1, out.shape[-1])
    r = ref.reshape(-1, ref.shape[-1])
    num = (o * r).sum(1)
    den = np.linalg.norm(o, axis=1) * np.linalg.norm(r, axis=1)
    cos = num[den > 0] / den[den > 0]
    assert cos.size == 0 or cos.min() >= MIN_COS, f"min cosine {cos.min():.7f}"


def fp16_vals(rng, *shape):
    return rng.standard_normal(shape).astype(np.float16).astype(np.float32)


def bf16_vals(rng, *shape):
    """N(0,1) values exactly representable in bf16 (as float32)."""
    return torch.from_numpy(rng.standard_normal(shape).astype(np.float32)).to(torch.bfloat16).float().numpy()


def gates_for(h, rng):
    return rng.uniform(0, 1, h).tolist()


PREFILL_CASES = [
    # n, s, h, h_kv, d, sparsity, sink, local
    (200, 200, 8, 2, 128, 0.5, 1, 2),      # ragged N (not a multiple of 64 / 256)
    (100, 300, 8, 2, 128, 0.5, 1, 2),      # history longer than the queries (attn.py:32-34)
    (320, 320, 4, 4, 128, 0.5, 1, 1),      # MHA (Llama-2 style group of 1)
    (256, 256, 8, 1, 128, 0.25, 2, 1),     # one KV head, group of 8
    (192, 192, 8, 2, 64, 0.5, 1, 2),       # head_dim 64
    (130, 130, 4, 2, 96, 0.5, 1, 1),       # head_dim 96 -> padded to 128 (scale uses 96)
    (640, 640, 8, 2, 128, 0.9, 1, 3),      # 7 of 8 heads streaming (one dense KV group)
    (1, 65, 4, 2, 128, 0.5, 1, 1),         # a single query row
]


@pytest.mark.parametrize("case", PREFILL_CASES)
def test_prefill_shapes_against_oracle(case):
    n, s, h, h_kv, d, sp, sink, local = case
    rng = np.random.default_rng(hash(case) % 2**32)
    q, k, v = fp16_vals(rng, n, h, d), fp16_vals(rng, s, h_kv, d), fp16_vals(rng, s, h_kv, d)
    gates = gates_for(h, rng)
    eng = sk.Engine(sk.EngineConfig(quant_bits=4, sink_blocks=sink, local_blocks=local, target_sparsity=sp),
                    sk.classify_heads(gates, sp, sink, local), device="cuda:0")
    out = eng.prefill(sk.Workload(q, k, v))
    ref_eng = O.OracleEngine(O.Config(quant_bits=4, sink_blocks=sink, local_blocks=local, target_sparsity=sp),
                             O.assign_roles(gates, sp, sink, local))
    ref = ref_eng.prefill(q, k, v)
    close(out, ref)
    assert {key: val for key, val in eng.ledger.tiles.items()} == ref_eng.tally.tiles


def test_prefill_bf16_inputs():
    rng = np.random.default_rng(5)
    n = s = 384
    h, h_kv, d = 8, 2, 128
    q, k, v = fp16_vals(rng, n, h, d), fp16_vals(rng, s, h_kv, d), fp16_vals(rng, s, h_kv, d)
    gates = gates_for(h, rng)
    qt, kt, vt = (torch.from_numpy(a).to(torch.bfloat16).cuda() for a in (q, k, v))
    eng = sk.Engine(sk.EngineConfig(), sk.classify_heads(gates, 0.5, 1, 2), device="cuda:0", dtype=torch.bfloat16)
    out = eng.prefill(sk.Workload(qt, kt, vt)).float().cpu().numpy()
    f = lambda t: t.float().cpu().numpy()  # noqa: E731  (the oracle sees the bf16-rounded values)
    ref = O.OracleEngine(O.Config(), O.assign_roles(gates, 0.5, 1, 2)).prefill(f(qt), f(kt), f(vt))
    close(out, ref, atol=3e-2)


DECODE_CASES = [
    # s, h, h_kv, d, bits, budget, sparsity, steps
    (2000, 4, 4, 128, 4, 512, 0.5, 6),       # MHA: streaming-only KV heads live in the ring pool
    (3000, 8, 1, 128, 4, 1024, 0.25, 6),     # group of 8 rows per KV head
    (1500, 8, 2, 64, 4, 512, 0.5, 6),        # head_dim 64
    (1100, 8, 2, 128, 8, 8192, 0.5, 4),      # budget >= pages: every page, no scoring
    (1100, 8, 2, 128, 4, 64, 0.5, 4),        # budget below the pins: pins only
    (700, 8, 2, 128, None, 256, 0.5, 5),     # fp16 pages
]


@pytest.mark.parametrize("case", DECODE_CASES)
def test_decode_shapes_against_oracle(case):
    s, h, h_kv, d, bits, budget, sp, steps = case
    rng = np.random.default_rng(abs(hash(case)) % 2**32)
    gates = gates_for(h, rng)
    k, v = fp16_vals(rng, s, h_kv, d), fp16_vals(rng, s, h_kv, d)
    cfg = sk.EngineConfig(quant_bits=bits, budget_tokens=budget, reuse_interval=2, local_blocks=2,
                          target_sparsity=sp)
    eng = sk.Engine(cfg, sk.classify_heads(gates, sp, 1, 2), device="cuda:0")
    eng.load_context(k, v)
    ref = O.OracleEngine(O.Config(quant_bits=bits, budget_tokens=budget, reuse_interval=2, local_blocks=2,
                                  target_sparsity=sp), O.assign_roles(gates, sp, 1, 2))
    ref.load_context(k, v)
    for t in range(steps):
        qn, kn, vn = fp16_vals(rng, h, d), fp16_vals(rng, h_kv, d), fp16_vals(rng, h_kv, d)
        res = eng.decode_step(qn, kn, vn)
        rr = ref.decode_step(qn, kn, vn)
        assert [tuple(tb.positions) for tb in res.index_tables] == rr.tables, f"step {t}"
        assert res.invoked == rr.invoked
        close(res.output, rr.output)
    assert eng.ledger.tiles == ref.tally.tiles


@pytest.mark.parametrize("s,steps", [(131072, 5), (262144, 5)])
def test_decode_128k_selection_and_outputs(s, steps):
    """BASELINE cfg2 / cfg3 geometry for one layer (32/8/128, 128k and 256k
    tokens, budget 4096, reuse 4, KV4, balanced gates): 5 decode steps (two
    selection steps) -- every index table bit-exact, outputs within tolerance."""
    rng = np.random.default_rng(128)
    h, h_kv, d = 32, 8, 128
    gates = [0.9 - 0.001 * i if i % 4 < 2 else 0.1 + 0.001 * i for i in range(h)]
    k, v = fp16_vals(rng, s, h_kv, d), fp16_vals(rng, s, h_kv, d)
    cfg = sk.EngineConfig(quant_bits=4, budget_tokens=4096, reuse_interval=4, local_blocks=4)
    eng = sk.Engine(cfg, sk.classify_heads(gates, 0.5, 1, 4), device="cuda:0")
    eng.load_context(k, v)
    ref = O.OracleEngine(O.Config(quant_bits=4, budget_tokens=4096, reuse_interval=4, local_blocks=4),
                         O.assign_roles(gates, 0.5, 1, 4))
    ref.load_context(k, v)
    del k, v
    for t in range(steps):
        qn, kn, vn = fp16_vals(rng, h, d), fp16_vals(rng, h_kv, d), fp16_vals(rng, h_kv, d)
        res = eng.decode_step(qn, kn, vn)
        rr = ref.decode_step(qn, kn, vn)
        assert [tuple(tb.positions) for tb in res.index_tables] == rr.tables, f"step {t}"
        close(res.output, rr.output)
    assert eng.ledger.selector_invocations == ref.tally.selector


def test_kv_head_shards_recombine_bitwise():
    """Two KV-head shards run as separate engines (what two ranks do) give,
    concatenated by head, exactly the unsharded engine's prefill and decode
    outputs: nothing in K1-K4 couples KV heads."""
    rng = np.random.default_rng(9)
    n = s = 512
    h, h_kv, d = 8, 4, 128
    gates = gates_for(h, rng)
    prof = sk.classify_heads(gates, 0.5, 1, 2)
    q, k, v = fp16_vals(rng, n, h, d), fp16_vals(rng, s, h_kv, d), fp16_vals(rng, s, h_kv, d)
    cfg = sk.EngineConfig(budget_tokens=256, reuse_interval=2)
    full = sk.Engine(cfg, prof, device="cuda:0")
    out_full = full.prefill(sk.Workload(q, k, v))
    shards = [shard_heads(h, h_kv, r, 2) for r in range(2)]
    engs = [sk.Engine(cfg, shard_profiles(prof, sh), device="cuda:0") for sh in shards]
    outs = [e.prefill(sk.Workload(*shard_prefill_inputs(q, k, v, sh))) for e, sh in zip(engs, shards)]
    np.testing.assert_array_equal(np.concatenate(outs, axis=1), out_full)
    for t in range(4):
        qn, kn, vn = fp16_vals(rng, h, d), fp16_vals(rng, h_kv, d), fp16_vals(rng, h_kv, d)
        rf = full.decode_step(qn, kn, vn)
        parts = [e.decode_step(*shard_decode_inputs(qn, kn, vn, sh)) for e, sh in zip(engs, shards)]
        np.testing.assert_array_equal(np.concatenate([p.output for p in parts], axis=0), rf.output)
        assert [tuple(tb.positions) for p in parts for tb in p.index_tables] == \
            [tuple(tb.positions) for tb in rf.index_tables]


@pytest.mark.parametrize("page,logical,bits", [(32, 16, 4), (128, 32, 4), (128, 16, 8), (32, 8, None)])
def test_other_page_geometries_against_oracle(page, logical, bits):
    """Physical pages of 32 / 128 tokens (the K4 plan falls back to explicit
    per-row masks for 64-row query tiles over non-64 key tiles), logical pages
    of 8-32 tokens: prefill outputs and ledgers, then decode index tables and
    outputs against the oracle."""
    rng = np.random.default_rng(page * 7 + logical)
    n = s = 520
    h, h_kv, d = 8, 2, 128
    gates = gates_for(h, rng)
    q, k, v = fp16_vals(rng, n, h, d), fp16_vals(rng, s, h_kv, d), fp16_vals(rng, s, h_kv, d)
    kw = dict(physical_page=page, logical_page=logical, quant_bits=bits, budget_tokens=4 * page, reuse_interval=2,
              local_blocks=2)
    eng = sk.Engine(sk.EngineConfig(**kw), sk.classify_heads(gates, 0.5, 1, 2), device="cuda:0")
    ref = O.OracleEngine(O.Config(**kw), O.assign_roles(gates, 0.5, 1, 2))
    close(eng.prefill(sk.Workload(q, k, v)), ref.prefill(q, k, v))
    for t in range(4):
        qn, kn, vn = fp16_vals(rng, h, d), fp16_vals(rng, h_kv, d), fp16_vals(rng, h_kv, d)
        res = eng.decode_step(qn, kn, vn)
        rr = ref.decode_step(qn, kn, vn)
        assert [tuple(tb.positions) for tb in res.index_tables] == rr.tables, f"step {t}"
        close(res.output, rr.output)
    assert eng.ledger.tiles == ref.tally.tiles


def test_decode_bf16_pool():
    rng = np.random.default_rng(77)
    s, h, h_kv, d = 1500, 8, 2, 128
    gates = gates_for(h, rng)
    cfg = sk.EngineConfig(quant_bits=4, budget_tokens=512, reuse_interval=2, local_blocks=2)
    kt = torch.from_numpy(fp16_vals(rng, s, h_kv, d)).to(torch.bfloat16)
    vt = torch.from_numpy(fp16_vals(rng, s, h_kv, d)).to(torch.bfloat16)
    eng = sk.Engine(cfg, sk.classify_heads(gates, 0.5, 1, 2), device="cuda:0", dtype=torch.bfloat16)
    eng.load_context(kt.cuda(), vt.cuda())
    ref = O.OracleEngine(O.Config(quant_bits=4, budget_tokens=512, reuse_interval=2, local_blocks=2),
                         O.assign_roles(gates, 0.5, 1, 2))
    ref.load_context(kt.float().numpy(), vt.float().numpy())
    for t in range(4):
        qn = torch.from_numpy(fp16_vals(rng, h, d)).to(torch.bfloat16)
        kn = torch.from_numpy(fp16_vals(rng, h_kv, d)).to(torch.bfloat16)
        vn = torch.from_numpy(fp16_vals(rng, h_kv, d)).to(torch.bfloat16)
        res = eng.decode_step(qn.cuda(), kn.cuda(), vn.cuda())
        rr = ref.decode_step(qn.float().numpy(), kn.float().numpy(), vn.float().numpy())
        assert [tuple(tb.positions) for tb in res.index_tables] == rr.tables, f"step {t}"
        close(res.output.float().cpu().numpy(), rr.output, atol=3e-2)


@pytest.mark.parametrize("n,pinned", [(1000, True), (300, False), (2048, True)])
def test_prefill_host_torch_equals_device_path(n, pinned):
    """Host torch inputs (pinned or pageable) give exactly the device-input
    path's output and ledger, and a non-finite host input raises."""
    rng = np.random.default_rng(n)
    h, h_kv, d = 8, 2, 128
    gates = gates_for(h, rng)
    prof = sk.classify_heads(gates, 0.5, 1, 2)
    q, k, v = (torch.from_numpy(fp16_vals(rng, *sh)).half() for sh in ((n, h, d), (n, h_kv, d), (n, h_kv, d)))
    if pinned:
        q, k, v = q.pin_memory(), k.pin_memory(), v.pin_memory()
    e_host = sk.Engine(sk.EngineConfig(), prof, device="cuda:0")
    e_dev = sk.Engine(sk.EngineConfig(), prof, device="cuda:0")
    out_h = e_host.prefill(sk.Workload(q, k, v))
    out_d = e_dev.prefill(sk.Workload(q.cuda(), k.cuda(), v.cuda()))
    torch.testing.assert_close(out_h, out_d, rtol=0, atol=0)
    assert e_host.ledger.tiles == e_dev.ledger.tiles
    assert e_host.cache.num_tokens == n
    q_bad = q.clone()
    q_bad[n // 3, 1, 5] = float("inf")
    with pytest.raises(ValueError, match="non-finite"):
        e_host.prefill(sk.Workload(q_bad, k, v))


@pytest.mark.parametrize("n", [5, 37, 300, 2049, 4096, 4097, 6144, 6145, 7000])
@pytest.mark.parametrize("ties", [False, True])
def test_topk_paths_against_oracle(n, ties):
    """K2's top-k -- the register path (n <= 6144 pages) and the staged
    fallback (n > 6144) -- against the oracle's (score desc, index asc)
    selection, on random and on heavily tied page scores."""
    from paper_2502_14866_b200.cache import PageStats, PhysicalPage

    rng = np.random.default_rng(n + 7 * ties)
    d = 16
    if ties:  # few distinct boxes -> many equal scores
        lo = rng.integers(-2, 1, (n, d)).astype(np.float64) * 0.5
        hi = lo + rng.integers(0, 2, (n, d)) * 0.5
    else:
        a, b = fp16_vals(rng, n, d).astype(np.float64), fp16_vals(rng, n, d).astype(np.float64)
        lo, hi = np.minimum(a, b), np.maximum(a, b)
    q = fp16_vals(rng, 2, d).astype(np.float64)
    z = np.zeros(d)
    ours_pages = [PhysicalPage(i, 0, 64, 64, None, None, z, z, z, z, [PageStats(lo[i], hi[i], 64)]) for i in range(n)]
    ref_pages = [O.Page(i, 64, None, None, None, None, None, None, [(lo[i], hi[i], 64)]) for i in range(n)]
    for k in sorted({4, 7, 64, max(4, n // 3), n - 1}):
        if k >= n:
            continue
        got = sk.select_pages(q, ours_pages, k * 64, 64)
        assert got == O.top_pages(q, ref_pages, k * 64, 64), (n, k, ties)


def test_inexact_wide_inputs_are_refused_not_rounded():
    """fp32/fp64 values the device dtype cannot hold would give page stats and
    selections that silently differ from the reference's; the boundary refuses
    them unless rounding is explicitly allowed."""
    rng = np.random.default_rng(3)
    x = rng.standard_normal((64, 16))  # fp64, not fp16-exact
    head = sk.cache.HeadPages(0, 64, 16, 4, True)
    with pytest.raises(ValueError, match="not exactly representable"):
        head.append(x, x)
    with pytest.raises(ValueError, match="not exactly representable"):
        sk.quantize_page(x, 4)
    with sk._device.rounding_allowed():
        codes, _, _ = sk.quantize_page(x, 4)
    assert codes.max() <= 15
    x16 = x.astype(np.float16).astype(np.float64)  # exact in fp16: accepted as is
    head.append(x16, x16)
    assert head.num_tokens == 64
