"""prefill_layers (host buffers, copies overlapped with the kernels) against
the sequential public API: same outputs bit for bit, same caches."""

import numpy as np
import pytest
import torch

import paper_2502_14866_b200 as sk

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d", [128, 96])
def test_pipelined_equals_sequential(d):
    torch.manual_seed(0)
    n_layers, n, h, hkv = 3, 1000, 8, 2
    gates = [0.9, 0.1, 0.8, 0.2, 0.85, 0.15, 0.7, 0.3]
    cfg = sk.EngineConfig(local_blocks=2)
    prof = sk.classify_heads(gates, 0.5, 1, 2)
    ins = [tuple(torch.randn(shape, dtype=torch.float16).pin_memory() for shape in ((n, h, d), (n, hkv, d), (n, hkv, d)))
           for _ in range(n_layers)]
    outs = [torch.empty((n, h, d), dtype=torch.float16).pin_memory() for _ in range(n_layers)]
    seq = [sk.Engine(cfg, prof, device="cuda:0") for _ in range(n_layers)]
    pip = [sk.Engine(cfg, prof, device="cuda:0") for _ in range(n_layers)]
    ref = [seq[i].prefill(sk.Workload(*ins[i])).cpu() for i in range(n_layers)]
    sk.prefill_layers(pip, ins, outs)
    for i in range(n_layers):
        assert torch.equal(outs[i], ref[i]), i
        for kv in range(hkv):
            a = seq[i].cache.pool_of(kv).live_pages()
            b = pip[i].cache.pool_of(kv).live_pages()
            assert [p.page_id for p in a] == [p.page_id for p in b]
            for pa, pb in zip(a, b):
                np.testing.assert_array_equal(pa.k_codes, pb.k_codes)
                np.testing.assert_array_equal(pa.v_codes, pb.v_codes)
    assert [e.ledger.tiles for e in seq] == [e.ledger.tiles for e in pip]


def test_pipelined_rejects_non_finite():
    cfg = sk.EngineConfig()
    prof = sk.classify_heads([0.9, 0.1], 0.5, 1, 2)
    q = torch.randn((100, 2, 64), dtype=torch.float16)
    k = torch.randn((100, 1, 64), dtype=torch.float16)
    v = k.clone()
    v[3, 0, 5] = float("nan")
    with pytest.raises(ValueError, match="non-finite"):
        sk.prefill_layers([sk.Engine(cfg, prof, device="cuda:0")] * 2, [(q, k, k), (q, k, v)],
                          [torch.empty_like(q), torch.empty_like(q)])


def test_reprefill_recycles_pool_like_a_fresh_engine():
    """A second (and third) prefill on the same Engine recycles its device
    pool (DevicePool.reset): outputs, pages and the following decode step
    must equal a fresh engine's -- shorter and longer contexts included."""
    rng = np.random.default_rng(5)
    h, hkv, d = 8, 2, 128
    gates = [0.9, 0.1, 0.8, 0.2, 0.85, 0.15, 0.7, 0.3]
    cfg = sk.EngineConfig(local_blocks=2, budget_tokens=256)
    prof = sk.classify_heads(gates, 0.5, 1, 2)
    reused = sk.Engine(cfg, prof, device="cuda:0")
    for n in (900, 333, 2100):
        q = rng.standard_normal((n, h, d)).astype(np.float16).astype(np.float32)
        k = rng.standard_normal((n, hkv, d)).astype(np.float16).astype(np.float32)
        v = rng.standard_normal((n, hkv, d)).astype(np.float16).astype(np.float32)
        fresh = sk.Engine(cfg, prof, device="cuda:0")
        a = reused.prefill(sk.Workload(q, k, v))
        b = fresh.prefill(sk.Workload(q, k, v))
        np.testing.assert_array_equal(a, b)
        for kv in range(hkv):
            pa, pb = reused.cache.pool_of(kv).live_pages(), fresh.cache.pool_of(kv).live_pages()
            assert [p.page_id for p in pa] == [p.page_id for p in pb]
            for x, y in zip(pa, pb):
                np.testing.assert_array_equal(x.k_codes, y.k_codes)
                np.testing.assert_array_equal(x.v_codes, y.v_codes)
                assert len(x.stats) == len(y.stats)
        qn = rng.standard_normal((h, d)).astype(np.float16).astype(np.float32)
        kn = rng.standard_normal((hkv, d)).astype(np.float16).astype(np.float32)
        vn = rng.standard_normal((hkv, d)).astype(np.float16).astype(np.float32)
        ra, rb = reused.decode_step(qn, kn, vn), fresh.decode_step(qn, kn, vn)
        assert [t.positions for t in ra.index_tables] == [t.positions for t in rb.index_tables]
        np.testing.assert_array_equal(ra.output, rb.output)
