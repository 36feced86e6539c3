"""One paged-K4 launch (sk_prefill_attn_paged) for ncu: cfg2 heads, a
SK_HIST-token KV4 history (default 32k) and a SK_CHUNK-token chunk (2k)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2502_14866_b200 as sk
from paper_2502_14866_b200.attn import run_prefill_paged

H, HKV, D = 32, 8, 128
s0, c = int(os.environ.get("SK_HIST", 32768)), int(os.environ.get("SK_CHUNK", 2048))
gates = [0.9 - 0.001 * i if i % 4 < 2 else 0.1 + 0.001 * i for i in range(H)]
eng = sk.Engine(sk.EngineConfig(quant_bits=4, local_blocks=4), sk.classify_heads(gates, 0.5, 1, 4), device="cuda:0",
                capacity_tokens=s0 + c)
g = torch.Generator(device="cuda").manual_seed(0)
eng.load_context(torch.randn((s0, HKV, D), generator=g, device="cuda", dtype=torch.float16),
                 torch.randn((s0, HKV, D), generator=g, device="cuda", dtype=torch.float16))
q = torch.randn((c, H, D), generator=g, device="cuda", dtype=torch.float16)
k = torch.randn((c, HKV, D), generator=g, device="cuda", dtype=torch.float16)
plan = eng._plan(c, s0 + c)
for _ in range(2):
    out = run_prefill_paged(eng.cache.pool, s0, q, k, k, plan, 1 / math.sqrt(D))
torch.cuda.synchronize()
print("done", float(out.float().abs().mean()))
