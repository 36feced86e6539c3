"""Phase timeline of the decode kernel (library built with -DSK_DECODE_TIMING)."""
import ctypes as C
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2502_14866_b200 as sk
from paper_2502_14866_b200 import _lib

ctx = 131072
H, HKV, D = 32, 8, 128
gates = [0.9 - 0.001 * h if h % 4 < 2 else 0.1 + 0.001 * h for h in range(H)]
cfg = sk.EngineConfig(quant_bits=4, budget_tokens=4096, reuse_interval=4, local_blocks=4)
e = sk.Engine(cfg, sk.classify_heads(gates, 0.5, 1, 4), device="cuda:0", capacity_tokens=ctx + 4096)
g = torch.Generator(device="cuda").manual_seed(0)
k = torch.randn((ctx + 5, HKV, D), generator=g, device="cuda", dtype=torch.float16)
e.load_context(k, k)
lib = _lib.load()
lib.sk_debug_decode_times.argtypes = [C.c_void_p]
for step in range(6):
    q = torch.randn((H, D), generator=g, device="cuda", dtype=torch.float16)
    e.decode_device(q, k[step], k[step + 1], D)
    torch.cuda.synchronize()
    buf = np.zeros((64, 10), np.uint64)
    assert lib.sk_debug_decode_times(buf.ctypes.data) == 0
    n = int((buf[:, 0] > 0).sum())
    t0 = buf[:n, 0].min()
    rel = (buf[:n].astype(np.int64) - int(t0)) / 1000.0
    rel[buf[:n] == 0] = np.nan
    print(f"step {step}: CTAs {n}; phase times (us, rel. to first CTA start) start/prologue/staged/items/merge/preticket/last/...")
    for i in range(0, n, max(1, n // 6)):
        print("  cta", i, np.round(rel[i, :9], 2))
    print("  max over CTAs", np.round(np.nanmax(rel[:, :9], axis=0), 2))
