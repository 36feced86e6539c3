"""Round-2 fixes on the B200 path, each against the oracle:

* K1 bulk appends that start inside the open page and end in a DIFFERENT
  partial page (the open page's CTA reads the staging page the last page
  refills; cache.py:211-251 semantics), over many streams at once;
* decode with streaming heads whose own (sink, local) window differs from
  the pool's (engine.py:264-267 attends streaming_schedule(profile));
* chunked prefill at physical_page=32 with streaming heads, where a 64-key
  K4 block mixes an attended page with an evicted one (the gathered history
  must be zero there, not recycled memory).
"""

import numpy as np
import pytest
import torch

import paper_2502_14866_b200 as sk
from oracle import sparsekv_oracle as O
from paper_2502_14866_b200 import _lib
from paper_2502_14866_b200.cache import DevicePool
from test_gpu_edges import fp16_vals
from test_gpu_parity import assert_close_attn

pytestmark = pytest.mark.gpu


def _assert_pages_equal(ours, theirs, with_stats=True):
    assert [p.page_id for p in ours] == [p.index for p in theirs]
    for po, pt in zip(ours, theirs):
        assert po.token_count == pt.tokens
        np.testing.assert_array_equal(po.k_codes, pt.k_codes[:pt.tokens].astype(po.k_codes.dtype))
        np.testing.assert_array_equal(po.v_codes, pt.v_codes[:pt.tokens].astype(po.v_codes.dtype))
        np.testing.assert_array_equal(po.k_scale, pt.k_scale)
        np.testing.assert_array_equal(po.k_zero, pt.k_zero)
        if with_stats:
            assert len(po.stats) == len(pt.bounds)
            for so, (kmin, kmax, cov) in zip(po.stats, pt.bounds):
                np.testing.assert_array_equal(so.k_min, kmin)
                np.testing.assert_array_equal(so.k_max, kmax)
                assert so.covered_tokens == cov


@pytest.mark.parametrize("bits", [4, 8, None])
def test_unaligned_bulk_appends_across_pages_many_streams(bits):
    """Every chunk starts mid-page and ends mid-page two or more pages later."""
    rng = np.random.default_rng(11)
    n_streams, d, page = 96, 128, 64
    chunks = [37, 150, 91, 200, 1, 63, 129, 70]
    pool = DevicePool([_lib.SK_KIND_DENSE] * (n_streams - 4) + [_lib.SK_KIND_STREAMING] * 4, d, page, 16, bits,
                      1, 2, device="cuda:0", capacity_tokens=64)  # small: forces growth too
    heads = [O.PagedHead(page, 16, bits, i < n_streams - 4, None if i < n_streams - 4 else (1, 2))
             for i in range(n_streams)]
    for m in chunks:
        k = fp16_vals(rng, n_streams, m, d)
        v = fp16_vals(rng, n_streams, m, d)
        kd = torch.from_numpy(k).to("cuda", torch.float16)
        vd = torch.from_numpy(v).to("cuda", torch.float16)
        pool.append(kd, vd, m * d, d, m)
        for i, h in enumerate(heads):
            h.append(k[i], v[i])
    for i in range(0, n_streams, 7):
        ours = pool.snapshot_pages(i, pool.live_indices(i), i)
        _assert_pages_equal(ours, heads[i].live(), with_stats=i < n_streams - 4)


def _engines(profiles, cfg_kw, oracle_roles):
    cfg = sk.EngineConfig(**cfg_kw)
    eng = sk.Engine(cfg, profiles, device="cuda:0")
    ref = O.OracleEngine(O.Config(**cfg_kw), oracle_roles)
    return eng, ref


@pytest.mark.parametrize("graph", [False, True])
def test_decode_honours_per_head_streaming_windows(graph):
    """Mixed groups (dense KV heads) whose streaming heads carry windows other
    than the config's: each row attends its own sink + local pages."""
    rng = np.random.default_rng(5)
    h, h_kv, d, s = 8, 2, 128, 64 * 40 + 17
    R, S = sk.RETRIEVAL, sk.STREAMING
    spec = [(R, 1, 2), (S, 3, 5), (S, 1, 1), (S, 2, 2), (R, 1, 2), (S, 4, 3), (R, 1, 2), (S, 1, 2)]
    profiles = [sk.HeadProfile(i, 0.9 if r == R else 0.1, r, sb, lb) for i, (r, sb, lb) in enumerate(spec)]
    roles = [O.Role(i, 0.9 if r == R else 0.1, r, sb, lb) for i, (r, sb, lb) in enumerate(spec)]
    kw = dict(quant_bits=4, budget_tokens=512, reuse_interval=2, sink_blocks=1, local_blocks=2)
    eng, ref = _engines(profiles, kw, roles)
    k, v = fp16_vals(rng, s, h_kv, d), fp16_vals(rng, s, h_kv, d)
    eng.load_context(k, v)
    ref.load_context(k, v)
    steps = [(fp16_vals(rng, h, d), fp16_vals(rng, h_kv, d), fp16_vals(rng, h_kv, d)) for _ in range(5)]
    if not graph:
        for t, (qn, kn, vn) in enumerate(steps):
            res = eng.decode_step(qn, kn, vn)
            rr = ref.decode_step(qn, kn, vn)
            assert [tuple(tb.positions) for tb in res.index_tables] == rr.tables, f"step {t}"
            assert_close_attn(res.output, rr.output)
        return
    from paper_2502_14866_b200.decode_graph import DecodeGraph
    dg = DecodeGraph([eng], max_steps=len(steps), head_dim=d)
    for t, (qn, kn, vn) in enumerate(steps):
        dg.q.copy_(torch.from_numpy(qn[None]))
        dg.k.copy_(torch.from_numpy(kn[None]))
        dg.v.copy_(torch.from_numpy(vn[None]))
        out = dg.step().float().cpu().numpy()[0]
        rr = ref.decode_step(qn, kn, vn)
        assert_close_attn(out, rr.output)


def test_streaming_pool_window_beyond_the_ring_is_refused():
    """A KV head whose whole group streams lives in the ring pool (sink+local
    pages of the config); a head asking for a wider window reads evicted
    pages, which the reference refuses too (page_at -> KeyError)."""
    rng = np.random.default_rng(6)
    h, h_kv, d, s = 4, 2, 64, 64 * 20
    R, S = sk.RETRIEVAL, sk.STREAMING
    profiles = [sk.HeadProfile(0, 0.9, R), sk.HeadProfile(1, 0.8, R),
                sk.HeadProfile(2, 0.1, S, 1, 2), sk.HeadProfile(3, 0.1, S, 1, 6)]
    eng = sk.Engine(sk.EngineConfig(quant_bits=4, sink_blocks=1, local_blocks=2), profiles, device="cuda:0")
    eng.load_context(fp16_vals(rng, s, h_kv, d), fp16_vals(rng, s, h_kv, d))
    with pytest.raises(KeyError, match="not resident"):
        eng.decode_step(fp16_vals(rng, h, d), fp16_vals(rng, h_kv, d), fp16_vals(rng, h_kv, d))


def test_chunked_prefill_page32_streaming_heads_zero_history():
    """physical_page 32: K4's 64-key blocks straddle a kept and an evicted page
    of the streaming ring; the gathered history is zero there.  The device
    memory the gather buffers come from is first filled with NaN."""
    rng = np.random.default_rng(9)
    h, h_kv, d, total, split = 8, 2, 128, 640, 450
    gates = [0.1, 0.2, 0.1, 0.05, 0.9, 0.1, 0.8, 0.2]  # KV head 0 all-streaming -> ring pool
    kw = dict(quant_bits=4, physical_page=32, logical_page=16, budget_tokens=256, reuse_interval=2,
              sink_blocks=1, local_blocks=3, tile_q_prefill=64)
    prof = sk.classify_heads(gates, 0.5, 1, 3)
    eng = sk.Engine(sk.EngineConfig(**kw), prof, device="cuda:0")
    ref = O.OracleEngine(O.Config(**kw), O.assign_roles(gates, 0.5, 1, 3))
    q, k, v = fp16_vals(rng, total, h, d), fp16_vals(rng, total, h_kv, d), fp16_vals(rng, total, h_kv, d)
    a = 0
    for b in (split, total):
        # poison the caching allocator's free blocks so uninitialised buffers hold NaN
        junk = torch.full((64 << 20,), float("nan"), dtype=torch.float16, device="cuda")
        del junk
        out = eng.prefill_chunk(sk.Workload(q[a:b], k[a:b], v[a:b]))
        rr = ref.prefill_chunk(q[a:b], k[a:b], v[a:b])
        assert np.isfinite(out).all()
        assert_close_attn(out, rr)
        a = b
    assert eng.ledger.tiles == ref.tally.tiles
