"""BASELINE cfg1 against the REAL reference's own run (tests/golden/make_cfg1.py,
sparsekv Engine.prefill + 256 x Engine.decode_step at 8k, 32/8 heads, D 128,
balanced 50% streaming, KV4, budget 4096, reuse 4; engine.py:136-286).

Bit-exact: the prefill and decode ledgers (142,176 / 264,192 and
282,624 / 1,068,928), the 512 selector calls, the per-(stage, head) tile
counts, every step's index tables and invoked flags, and the final pages of
every KV head (codes, scale/zero, logical-page stats).  Within the
north_star tolerance (max-abs 2e-2, per-head cosine >= 0.9999): prefill
outputs at 256 sampled rows and every decode output -- through the eager
Engine and through the CUDA-graph decode step the bench times."""

import os
import sys

import numpy as np
import pytest
import torch

import paper_2502_14866_b200 as sk
from test_gpu_parity import assert_close_attn

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
import make_cfg1 as G  # noqa: E402

pytestmark = pytest.mark.gpu
FIX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfg1_ref.npz")


@pytest.fixture(scope="module")
def case():
    g = dict(np.load(FIX))
    arrays = G.inputs()
    assert G.input_digest(arrays) == str(g["input_sha256"]), "regenerated inputs differ from the reference run's"
    return g, arrays


def _engine():
    cfg = sk.EngineConfig(**G.CFG)
    prof = sk.classify_heads(G.balanced_gates(), cfg.target_sparsity, cfg.sink_blocks, cfg.local_blocks)
    return sk.Engine(cfg, prof, device="cuda:0")


def _check_prefill(g, out):
    assert_close_attn(out[g["sample_rows"]], g["prefill_rows"])
    o = out.astype(np.float64)
    np.testing.assert_allclose(o.sum(axis=(0, 2)), g["prefill_head_sum"], rtol=0, atol=2e-2 * o.shape[0])
    np.testing.assert_allclose((o ** 2).sum(axis=(0, 2)), g["prefill_head_sumsq"], rtol=2e-3)


def _check_ledger(g, eng):
    assert (eng.ledger.visited("prefill"), eng.ledger.total("prefill")) == tuple(g["ledger_prefill"])
    assert (eng.ledger.visited("decode"), eng.ledger.total("decode")) == tuple(g["ledger_decode"])
    tiles = {f"{st}:{h}": list(v) for (st, h), v in eng.ledger.tiles.items()}
    assert tiles == {k: list(v) for k, v in zip(g["tile_keys"], g["tile_vals"])}
    assert [eng.ledger.selector_invocations.get(kv, 0) for kv in range(G.HKV)] == list(g["selector_calls"])


def test_cfg1_eager_engine_matches_reference_run(case):
    g, (q, k, v, qn, kn, vn) = case
    eng = _engine()
    _check_prefill(g, eng.prefill(sk.Workload(q, k, v)))
    for t in range(G.STEPS):
        res = eng.decode_step(qn[t], kn[t], vn[t])
        ref_tables = [tuple(int(x) for x in row if x >= 0) for row in g["tables"][t]]
        assert [tuple(tb.positions) for tb in res.index_tables] == ref_tables, f"step {t} index tables"
        assert {kv: int(r) for kv, r in res.invoked.items()} == \
            {kv: int(g["invoked"][t, kv]) for kv in res.invoked}, f"step {t} invoked"
        assert_close_attn(res.output, g["decode_out"][t].astype(np.float32))
    _check_ledger(g, eng)
    digests = [G.page_digest(eng.cache.pool_of(kv).live_pages()) for kv in range(G.HKV)]
    assert digests == list(g["page_digests"]), "final KV4 pages differ from the reference's"


def test_cfg1_graph_decode_matches_reference_run(case):
    from paper_2502_14866_b200.decode_graph import DecodeGraph
    g, (q, k, v, qn, kn, vn) = case
    eng = _engine()
    eng.prefill_device(*(torch.from_numpy(a).to("cuda", torch.float16) for a in (q, k, v)), G.D)
    dg = DecodeGraph([eng], max_steps=G.STEPS, head_dim=G.D)
    for t in range(G.STEPS):
        dg.q.copy_(torch.from_numpy(qn[t][None]))
        dg.k.copy_(torch.from_numpy(kn[t][None]))
        dg.v.copy_(torch.from_numpy(vn[t][None]))
        out = dg.step().float().cpu().numpy()[0]
        assert_close_attn(out, g["decode_out"][t].astype(np.float32))
    _check_ledger(g, eng)
    digests = [G.page_digest(eng.cache.pool_of(kv).live_pages()) for kv in range(G.HKV)]
    assert digests == list(g["page_digests"])
