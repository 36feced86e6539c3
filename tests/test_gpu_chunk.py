"""Continued (chunked) prefill on the B200: K1b pool gather + K4 over the
(cached history ++ chunk) + K1 append, against OracleEngine.prefill_chunk
(tests/test_chunk_oracle.py pins its semantics on CPU).  Outputs within the
north_star tolerance; page codes / stats and the following decode step's
selections bit-exact."""

import numpy as np
import pytest
import torch

import paper_2502_14866_b200 as sk
from oracle import sparsekv_oracle as O
from test_gpu_parity import assert_close_attn
from test_gpu_edges import bf16_vals, fp16_vals

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("bits,dtype", [(4, torch.float16), (8, torch.float16), (None, torch.float16),
                                        (4, torch.bfloat16)])
def test_gather_is_snapshot_dequantised(bits, dtype):
    rng = np.random.default_rng(7)
    s, h_kv, d = 1000, 3, 128
    gates = [0.9, 0.1, 0.1, 0.1, 0.8, 0.2]  # KV head 1 all-streaming (ring), 0 and 2 dense
    cfg = sk.EngineConfig(quant_bits=bits, local_blocks=3)
    eng = sk.Engine(cfg, sk.classify_heads(gates, 0.5, 1, 3), dtype=dtype, device="cuda:0")
    vals = fp16_vals if dtype == torch.float16 else bf16_vals
    eng.load_context(vals(rng, s, h_kv, d), vals(rng, s, h_kv, d))
    pool = eng.cache.pool
    kg, vg = pool.gather()
    kg, vg = kg.float().cpu().numpy(), vg.float().cpu().numpy()
    ulp = 2.0 ** (-10 if dtype == torch.float16 else -7)
    for kv in range(h_kv):
        pages = pool.snapshot_pages(kv, pool.live_indices(kv), kv)
        assert len(pages) == (16 if kv != 1 else 4)
        for pg in pages:
            kk, vv = pg.dequantize()
            sl = slice(pg.page_id * 64, pg.page_id * 64 + pg.token_count)
            np.testing.assert_allclose(kg[sl, kv], kk, rtol=ulp, atol=1e-5, err_msg=f"K page {pg.page_id}")
            np.testing.assert_allclose(vg[sl, kv], vv, rtol=ulp, atol=1e-5, err_msg=f"V page {pg.page_id}")


CHUNK_CASES = [
    # (splits, total, H, Hkv, bits, sparsity)
    ((256,), 700, 8, 2, 4, 0.5),
    ((100, 357), 600, 8, 2, 4, 0.5),        # unaligned chunk starts, partial open pages
    ((64, 128, 200), 333, 4, 4, 8, 0.25),   # MHA, 8-bit pages
    ((300,), 520, 8, 2, None, 0.5),         # fp16 pages
]


@pytest.mark.parametrize("paged", [False, True], ids=["gather", "paged"])
@pytest.mark.parametrize("case", CHUNK_CASES)
def test_chunked_prefill_against_oracle(case, paged):
    splits, total, h, h_kv, bits, sp = case
    rng = np.random.default_rng(sum(splits) + total)
    d = 128
    gates = list(rng.uniform(0, 1, h))
    q, k, v = fp16_vals(rng, total, h, d), fp16_vals(rng, total, h_kv, d), fp16_vals(rng, total, h_kv, d)
    cfg = sk.EngineConfig(quant_bits=bits, budget_tokens=256, reuse_interval=2, local_blocks=2, target_sparsity=sp)
    eng = sk.Engine(cfg, sk.classify_heads(gates, sp, 1, 2), device="cuda:0", paged_history=paged)
    ref = O.OracleEngine(O.Config(quant_bits=bits, budget_tokens=256, reuse_interval=2, local_blocks=2,
                                  target_sparsity=sp), O.assign_roles(gates, sp, 1, 2))
    a = 0
    for b in list(splits) + [total]:
        w = sk.Workload(q[a:b], k[a:b], v[a:b])
        out = eng.prefill_chunk(w)
        rr = ref.prefill_chunk(q[a:b], k[a:b], v[a:b])
        assert_close_attn(out, rr)
        a = b
    assert eng.ledger.tiles == ref.tally.tiles
    for kv in range(h_kv):  # the appended pages are the reference's, bit for bit
        ours = eng.cache.pool_of(kv).live_pages()
        theirs = ref.pools.head(kv).live()
        assert [p.page_id for p in ours] == [p.index for p in theirs]
        for po, pt in zip(ours, theirs):
            np.testing.assert_array_equal(po.k_codes, pt.k_codes[:pt.tokens].astype(po.k_codes.dtype))
            np.testing.assert_array_equal(po.v_codes, pt.v_codes[:pt.tokens].astype(po.v_codes.dtype))
    for t in range(3):  # decode continues from the chunked cache with the reference's selections
        qn, kn, vn = fp16_vals(rng, h, d), fp16_vals(rng, h_kv, d), fp16_vals(rng, h_kv, d)
        res = eng.decode_step(qn, kn, vn)
        rr = ref.decode_step(qn, kn, vn)
        assert [tuple(tb.positions) for tb in res.index_tables] == rr.tables, f"step {t}"
        assert_close_attn(res.output, rr.output)


def test_chunked_prefill_32k_matches_one_shot():
    """cfg2 head geometry (32 Q / 8 KV heads, D 128), 32k context as eight 4k
    chunks over fp16 pages vs one 32k prefill: the same attention up to
    accumulation order (no oracle at this size)."""
    torch.manual_seed(0)
    s, h, h_kv, d, c = 32768, 32, 8, 128, 4096
    gates = [0.9 - 0.01 * i if i % 4 < 2 else 0.1 + 0.01 * i for i in range(h)]
    cfg = sk.EngineConfig(quant_bits=None, local_blocks=4)
    prof = sk.classify_heads(gates, 0.5, 1, 4)
    q = torch.randn((s, h, d), device="cuda", dtype=torch.float16)
    k = torch.randn((s, h_kv, d), device="cuda", dtype=torch.float16)
    v = torch.randn((s, h_kv, d), device="cuda", dtype=torch.float16)
    one = sk.Engine(cfg, prof, device="cuda:0").prefill_device(q, k, v, d)
    eng = sk.Engine(cfg, prof, device="cuda:0", capacity_tokens=s)
    outs = [eng.prefill_chunk_device(q[a:a + c], k[a:a + c], v[a:a + c], d) for a in range(0, s, c)]
    got = torch.cat(outs).float()
    err = (got - one.float()).abs().max().item()
    cos = torch.nn.functional.cosine_similarity(got.transpose(0, 1).reshape(h, -1),
                                                one.float().transpose(0, 1).reshape(h, -1), dim=1).min().item()
    assert err <= 2e-2 and cos >= 0.9999, (err, cos)
    assert eng.cache.num_tokens == s


@pytest.mark.parametrize("page,hist,chunk,dtype", [(64, 4096 + 17, 333, torch.float16), (32, 2048 + 40, 100, torch.float16),
                                                   (64, 3000, 600, torch.bfloat16)])
def test_paged_k4_equals_gathered_history(page, hist, chunk, dtype):
    """K4 reading the KV4 history through the page table (sk_prefill_attn_paged)
    gives the outputs of K4 over the K1b-expanded history, to fp rounding of
    the accumulation order (same dequantised values, same schedules)."""
    import math

    from paper_2502_14866_b200.attn import run_prefill, run_prefill_paged
    h, h_kv, d = 8, 2, 128
    gates = [0.9, 0.1, 0.8, 0.2, 0.05, 0.15, 0.7, 0.6]
    cfg = sk.EngineConfig(physical_page=page, logical_page=16, quant_bits=4, sink_blocks=1, local_blocks=2)
    eng = sk.Engine(cfg, sk.classify_heads(gates, 0.5, 1, 2), device="cuda:0", dtype=dtype,
                    capacity_tokens=hist + chunk)
    g = torch.Generator(device="cuda").manual_seed(page + hist)
    eng.load_context(torch.randn((hist, h_kv, d), generator=g, device="cuda").to(dtype),
                     torch.randn((hist, h_kv, d), generator=g, device="cuda").to(dtype))
    q = torch.randn((chunk, h, d), generator=g, device="cuda").to(dtype)
    k = torch.randn((chunk, h_kv, d), generator=g, device="cuda").to(dtype)
    v = torch.randn((chunk, h_kv, d), generator=g, device="cuda").to(dtype)
    pool = eng.cache.pool
    plan = eng._plan(chunk, hist + chunk)
    kf, vf = pool.gather(extra_tokens=chunk)
    kf[hist:], vf[hist:] = k, v
    ref = run_prefill(q, kf, vf, plan, 1 / math.sqrt(d)).float()
    out = run_prefill_paged(pool, hist, q, k, v, plan, 1 / math.sqrt(d)).float()
    assert torch.isfinite(out).all()
    assert (out - ref).abs().max().item() <= (2e-3 if dtype == torch.float16 else 1.6e-2)
