"""Cache snapshot round trip on the device pools (cache.py:333-413,
SURVEY 8(f) item 2): dump_jsonl -> TwoWayCache.load_jsonl -> dump_jsonl is
byte-identical, restored pages (codes, scale/zero, logical stats, token
counts) equal the originals, and a restored partial page refuses appends
with the reference's error."""

import io
import os
import sys

import numpy as np
import pytest

import paper_2502_14866_b200 as sk

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("bits", [4, 8, None])
def test_snapshot_round_trip(bits):
    rng = np.random.default_rng(40 + (bits or 0))
    s, h, h_kv, d = 700, 8, 2, 128
    gates = [0.9, 0.1, 0.8, 0.2, 0.05, 0.15, 0.12, 0.11]  # kv 1 all-streaming -> streaming pool
    k = rng.standard_normal((s, h_kv, d)).astype(np.float16).astype(np.float32)
    v = rng.standard_normal((s, h_kv, d)).astype(np.float16).astype(np.float32)
    k[:, 0, 5] = 0.25  # a constant channel (scale forced to 1)
    eng = sk.Engine(sk.EngineConfig(quant_bits=bits, local_blocks=2), sk.classify_heads(gates, 0.75, 1, 2),
                    device="cuda:0")
    eng.load_context(k, v)
    buf = io.StringIO()
    eng.cache.dump_jsonl(buf)
    text = buf.getvalue()
    restored = sk.TwoWayCache.load_jsonl(io.StringIO(text), device="cuda:0")
    buf2 = io.StringIO()
    restored.dump_jsonl(buf2)
    assert buf2.getvalue() == text
    assert restored.num_tokens == s
    assert sorted(restored.dense_pool) == sorted(eng.cache.dense_pool)
    assert sorted(restored.streaming_pool) == sorted(eng.cache.streaming_pool)
    with pytest.raises(ValueError, match="partial page restored|restored from a snapshot"):
        restored.append_tokens(0, k[:1, 0], v[:1, 0])


# ---- interop with snapshots the reference itself wrote (tests/golden/make_snapshot.py) ----------
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("bits,name", [(4, "snapshot_ref_kv4.jsonl"), (None, "snapshot_ref_fp16.jsonl")])
def test_reference_snapshot_loads_and_dumps_back_identically(bits, name):
    """A JSONL snapshot written by the reference (cache.py:333-345) loads into
    the device pools and dumps back byte for byte."""
    text = open(f"{GOLDEN}/{name}").read()
    restored = sk.TwoWayCache.load_jsonl(io.StringIO(text), device="cuda:0")
    buf = io.StringIO()
    restored.dump_jsonl(buf)
    assert buf.getvalue() == text


@pytest.mark.parametrize("bits,name", [(4, "snapshot_ref_kv4.jsonl"), (None, "snapshot_ref_fp16.jsonl")])
def test_same_appends_dump_what_the_reference_dumps(bits, name):
    """The same appends (uneven chunks: an open partial page, streaming
    evictions) through the device pools dump the reference's bytes."""
    sys.path.insert(0, GOLDEN)
    from snapshot_inputs import CHUNKS as chunks, inputs
    k, v = inputs()
    c = sk.TwoWayCache(64, 16, bits, dense_heads=[0, 2], streaming_heads=[1], sink_blocks=1, local_blocks=2,
                       device="cuda:0", capacity_tokens=k.shape[0])
    t = 0
    for m in chunks:
        for h in range(3):
            c.append_tokens(h, k[t:t + m, h], v[t:t + m, h])
        t += m
    buf = io.StringIO()
    c.dump_jsonl(buf)
    assert buf.getvalue() == open(f"{GOLDEN}/{name}").read()
