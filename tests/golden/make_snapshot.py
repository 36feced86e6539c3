"""Reference-made JSONL snapshots (TwoWayCache.dump_jsonl, reference
cache.py:333-345) for tests/test_gpu_snapshot.py's interop checks.  Run in
the container that holds /root/reference:

    python tests/golden/make_snapshot.py

Two caches (KV4 and raw fp16 pages), dense heads 0, 2 and streaming head 1,
on the inputs of snapshot_inputs.py."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from snapshot_inputs import CHUNKS, inputs  # noqa: E402
from sparsekv.cache import TwoWayCache  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def build(bits):
    k, v = inputs()
    c = TwoWayCache(64, 16, bits, dense_heads=[0, 2], streaming_heads=[1], sink_blocks=1, local_blocks=2)
    t = 0
    for m in CHUNKS:
        for h in range(3):
            c.append_tokens(h, k[t:t + m, h], v[t:t + m, h])
        t += m
    return c


if __name__ == "__main__":
    for bits, name in ((4, "snapshot_ref_kv4.jsonl"), (None, "snapshot_ref_fp16.jsonl")):
        with open(os.path.join(HERE, name), "w") as fp:
            build(bits).dump_jsonl(fp)
        print("wrote", name)
