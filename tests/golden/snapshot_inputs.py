"""Inputs of the reference-made snapshot fixtures (make_snapshot.py) and of
the device-side replay in tests/test_gpu_snapshot.py: fp16-valued K/V for
KV heads 0-2 (D = 16) appended in uneven chunks, so the dumps hold an open
partial page and streaming evictions."""
import numpy as np

CHUNKS = (70, 1, 64, 37, 28)


def inputs(seed=11, n=200, d=16, heads=3):
    rng = np.random.default_rng(seed)
    k = rng.standard_normal((n, heads, d)).astype(np.float16).astype(np.float32)
    v = rng.standard_normal((n, heads, d)).astype(np.float16).astype(np.float32)
    return k, v
