"""Short representative workload for ncu: one 128k-context layer prefill
(K4 + K1) and 8 eager decode steps (K2 on steps 0 and 4, K3 fused)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2502_14866_b200 as sk

ctx = int(os.environ.get("SK_CTX", 131072))
H, HKV, D = 32, 8, 128
gates = [0.9 - 0.001 * h if h % 4 < 2 else 0.1 + 0.001 * h for h in range(H)]
cfg = sk.EngineConfig(quant_bits=4, budget_tokens=4096, reuse_interval=4, local_blocks=4)
prof = sk.classify_heads(gates, 0.5, 1, 4)
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn((ctx, H, D), generator=g, device="cuda", dtype=torch.float16)
k = torch.randn((ctx, HKV, D), generator=g, device="cuda", dtype=torch.float16)
v = torch.randn((ctx, HKV, D), generator=g, device="cuda", dtype=torch.float16)
eng = sk.Engine(cfg, prof, device="cuda:0", capacity_tokens=ctx + 64)
eng.prefill_device(q, k, v, D)
for t in range(8):
    qn = torch.randn((H, D), generator=g, device="cuda", dtype=torch.float16)
    kn = torch.randn((HKV, D), generator=g, device="cuda", dtype=torch.float16)
    eng.decode_device(qn, kn, kn.clone(), D)
torch.cuda.synchronize()
print("done", eng.cache.num_tokens)
