"""Batched decode (BASELINE cfg4 extension): B sequences in one device pool
per layer, decoded by one CUDA-graph step, must reproduce each sequence's
own Engine.decode_step (selections -> identical pages -> same outputs)."""

import numpy as np
import pytest
import torch

import paper_2502_14866_b200 as sk
from paper_2502_14866_b200.batch import BatchedLayer
from paper_2502_14866_b200.decode_graph import DecodeGraph

pytestmark = pytest.mark.gpu


def test_batched_graph_matches_per_sequence_engines():
    rng = np.random.default_rng(31)
    B, s, h, h_kv, d, L = 3, 2048 + 21, 8, 2, 128, 2
    gates = [0.9, 0.8, 0.1, 0.2, 0.85, 0.15, 0.12, 0.11]
    cfg = sk.EngineConfig(quant_bits=4, budget_tokens=512, reuse_interval=3, local_blocks=4)
    prof = sk.classify_heads(gates, 0.5, 1, 4)
    hist = [[(rng.standard_normal((s, h_kv, d)).astype(np.float16), rng.standard_normal((s, h_kv, d)).astype(np.float16))
             for _ in range(B)] for _ in range(L)]
    layers = [BatchedLayer(cfg, prof, B, h_kv, d, device="cuda:0", capacity_tokens=s + 64) for _ in range(L)]
    eng = [[sk.Engine(cfg, prof, device="cuda:0") for _ in range(B)] for _ in range(L)]
    for li in range(L):
        for b in range(B):
            k, v = hist[li][b]
            layers[li].load_context(b, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
            eng[li][b].load_context(k.astype(np.float32), v.astype(np.float32))
    dg = DecodeGraph(layers, 16, d, record_ledger=False)
    for t in range(7):
        q = rng.standard_normal((L, B, h, d)).astype(np.float16)
        kn = rng.standard_normal((L, B, h_kv, d)).astype(np.float16)
        vn = rng.standard_normal((L, B, h_kv, d)).astype(np.float16)
        dg.q.copy_(torch.from_numpy(q.reshape(L, B * h, d)))
        dg.k.copy_(torch.from_numpy(kn.reshape(L, B * h_kv, d)))
        dg.v.copy_(torch.from_numpy(vn.reshape(L, B * h_kv, d)))
        out = dg.step().float().cpu().numpy().reshape(L, B, h, d)
        for li in range(L):
            for b in range(B):
                res = eng[li][b].decode_step(q[li, b].astype(np.float32), kn[li, b].astype(np.float32),
                                             vn[li, b].astype(np.float32))
                np.testing.assert_allclose(out[li, b], res.output, atol=2e-3, rtol=0, err_msg=f"step {t} layer {li} seq {b}")
    assert all(p.tokens_host == [s + 7] * (B * h_kv) for p in (ly.pool for ly in layers))


@pytest.mark.parametrize("batch,h,h_kv", [(40, 8, 1), (12, 32, 8), (5, 8, 2)])
def test_batched_eager_matches_engines_all_cluster_sizes(batch, h, h_kv):
    """40 / 96 / 10 streams exercise the 1-, 2- and 8-CTA decode layouts
    (cluster_for in decode.cu): each sequence's output must match its own
    Engine.  Covers every output row and channel of the cluster merge."""
    rng = np.random.default_rng(batch)
    s, d = 1200 + batch, 128
    gates = rng.uniform(0, 1, h).tolist()
    cfg = sk.EngineConfig(quant_bits=4, budget_tokens=256, reuse_interval=2, local_blocks=2)
    prof = sk.classify_heads(gates, 0.5, 1, 2)
    layer = BatchedLayer(cfg, prof, batch, h_kv, d, device="cuda:0", capacity_tokens=s + 32)
    engs = []
    for b in range(batch):
        k = rng.standard_normal((s, h_kv, d)).astype(np.float16)
        v = rng.standard_normal((s, h_kv, d)).astype(np.float16)
        layer.load_context(b, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
        e = sk.Engine(cfg, prof, device="cuda:0")
        e.load_context(k.astype(np.float32), v.astype(np.float32))
        engs.append(e)
    dg = DecodeGraph([layer], 8, d, record_ledger=False)
    for t in range(3):
        q = rng.standard_normal((batch, h, d)).astype(np.float16)
        kn = rng.standard_normal((batch, h_kv, d)).astype(np.float16)
        vn = rng.standard_normal((batch, h_kv, d)).astype(np.float16)
        dg.q.copy_(torch.from_numpy(q.reshape(1, batch * h, d)))
        dg.k.copy_(torch.from_numpy(kn.reshape(1, batch * h_kv, d)))
        dg.v.copy_(torch.from_numpy(vn.reshape(1, batch * h_kv, d)))
        out = dg.step().float().cpu().numpy().reshape(batch, h, d)
        for b in range(batch):
            res = engs[b].decode_step(q[b].astype(np.float32), kn[b].astype(np.float32), vn[b].astype(np.float32))
            np.testing.assert_allclose(out[b], res.output, atol=2e-3, rtol=0, err_msg=f"step {t} seq {b}")


RAGGED = {
    "cfg4_6seq": [4100, 9000, 12037, 6500, 16384, 5000],       # 48 streams: K3 splits each over CTAs
    "cfg4_12seq": [4100, 9000, 5037, 6500, 8192, 5000, 4097, 7001, 4300, 6100, 5555, 4444],  # 96: one CTA
}                                                                # per stream, pages staged in smem


@pytest.mark.parametrize("lens", list(RAGGED.values()), ids=list(RAGGED))
def test_ragged_cfg4_batch_against_oracle(lens):
    """BASELINE cfg4 geometry (32 Q / 8 KV heads, D 128, balanced gates, KV4,
    budget 4096, reuse 4) for a RAGGED batch: every sequence has its own
    context length, page-table rows and token counts in one pool.  Each
    sequence is checked against its own OracleEngine (not the repo's Engine):
    the K2 selection of every stream bit-exact on every step, outputs within
    the north_star tolerance."""
    from oracle import sparsekv_oracle as O
    from test_gpu_parity import assert_close_attn
    rng = np.random.default_rng(4)
    h, h_kv, d = 32, 8, 128
    B = len(lens)
    gates = [0.9 - 0.001 * i if i % 4 < 2 else 0.1 + 0.001 * i for i in range(h)]
    kw = dict(quant_bits=4, budget_tokens=4096, reuse_interval=4, local_blocks=4)
    cfg = sk.EngineConfig(**kw)
    prof = sk.classify_heads(gates, 0.5, 1, 4)
    layer = BatchedLayer(cfg, prof, B, h_kv, d, device="cuda:0", capacity_tokens=max(lens) + 64)
    refs = []
    f16 = lambda *s: rng.standard_normal(s).astype(np.float16)  # noqa: E731
    for b, s in enumerate(lens):
        k, v = f16(s, h_kv, d), f16(s, h_kv, d)
        layer.load_context(b, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
        r = O.OracleEngine(O.Config(**kw), O.assign_roles(gates, 0.5, 1, 4))
        r.load_context(k.astype(np.float32), v.astype(np.float32))
        refs.append(r)
    steps = 6
    dg = DecodeGraph([layer], steps, d, record_ledger=False)
    for t in range(steps):
        q, kn, vn = f16(B, h, d), f16(B, h_kv, d), f16(B, h_kv, d)
        dg.q.copy_(torch.from_numpy(q.reshape(1, B * h, d)))
        dg.k.copy_(torch.from_numpy(kn.reshape(1, B * h_kv, d)))
        dg.v.copy_(torch.from_numpy(vn.reshape(1, B * h_kv, d)))
        out = dg.step().float().cpu().numpy().reshape(B, h, d)
        sel = dg.sel[0].cpu().numpy()
        cnt = dg.cnt[0].cpu().numpy()
        for b in range(B):
            rr = refs[b].decode_step(q[b].astype(np.float32), kn[b].astype(np.float32), vn[b].astype(np.float32))
            for kv in range(h_kv):
                st = b * h_kv + kv
                assert tuple(sel[st, :cnt[st]]) == rr.tables[kv * 4], f"step {t} seq {b} kv {kv}"
            assert_close_attn(out[b], rr.output)
    assert [layer.pool.tokens_host[b * h_kv] for b in range(B)] == [s + steps for s in lens]
