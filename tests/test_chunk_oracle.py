"""Continued (chunked) prefill in the oracle (CPU).  The reference has no
chunked entry point; OracleEngine.prefill_chunk composes its pinned pieces
(dequantised history as the decode path reads it + the static prefill
schedules).  Known answers: with raw pages (quant_bits None) and chunk
boundaries on tile edges, chunked prefill reproduces one-shot prefill
bit-for-bit, rows, tallies and cache alike."""

import numpy as np
import pytest

from oracle import sparsekv_oracle as O


def _inputs(s, h, h_kv, d, seed=0):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((s, h, d)).astype(np.float32), rng.standard_normal((s, h_kv, d)).astype(np.float32),
            rng.standard_normal((s, h_kv, d)).astype(np.float32))


@pytest.mark.parametrize("splits", [(128,), (64, 192), (64, 128, 256, 320)])
def test_raw_chunks_equal_one_shot(splits):
    q, k, v = _inputs(333, 4, 2, 32)
    roles = O.assign_roles([0.9, 0.1, 0.2, 0.3], 0.5, 1, 2)  # KV head 1 is all-streaming
    cfg = O.Config(quant_bits=None)
    one = O.OracleEngine(cfg, roles)
    full = one.prefill(q, k, v)
    ch = O.OracleEngine(cfg, roles)
    outs, a = [], 0
    for b in list(splits) + [q.shape[0]]:
        outs.append(ch.prefill_chunk(q[a:b], k[a:b], v[a:b]))
        a = b
    np.testing.assert_array_equal(np.concatenate(outs), full)
    assert ch.pools.num_tokens == one.pools.num_tokens
    for kv in range(2):
        assert sorted(ch.pools.head(kv).pages) == sorted(one.pools.head(kv).pages)
    # the ledger differs only by the per-chunk totals: visited tiles are the same
    assert ch.tally.visited() == one.tally.visited()


def test_quantised_history_is_what_decode_reads():
    """A one-token chunk on a dense head attends every page dequantised in
    the q dtype plus the raw token: exactly a decode step whose selection
    keeps every page (budget >= context)."""
    q, k, v = _inputs(200, 2, 1, 32, seed=3)
    roles = O.assign_roles([0.9, 0.8], 0.0, 1, 2)
    cfg = O.Config(quant_bits=4, budget_tokens=4096)
    a, b = O.OracleEngine(cfg, roles), O.OracleEngine(cfg, roles)
    a.load_context(k[:199], v[:199])
    b.load_context(k[:199], v[:199])
    out_chunk = a.prefill_chunk(q[199:], k[199:], v[199:])[0]
    out_dec = b.decode_step(q[199], k[199], v[199]).output
    np.testing.assert_allclose(out_chunk, out_dec, rtol=0, atol=1e-6)


def test_window_beyond_ring_raises():
    q, k, v = _inputs(400, 2, 1, 32, seed=5)
    roles = [O.Role(0, 0.1, O.STREAMING, 1, 4), O.Role(1, 0.2, O.STREAMING, 1, 4)]
    eng = O.OracleEngine(O.Config(quant_bits=4, local_blocks=2), roles)
    eng.load_context(k[:320], v[:320])
    with pytest.raises(ValueError, match="evicted"):
        eng.prefill_chunk(q[320:], k[320:], v[320:])
