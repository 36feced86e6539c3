"""cfg4 workload for ncu: 16 sequences x 64k context, one layer, 8 decode
steps through the CUDA-graph runner (K2 on steps 0 and 4)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2502_14866_b200 as sk
from paper_2502_14866_b200.batch import BatchedLayer
from paper_2502_14866_b200.decode_graph import DecodeGraph

B, ctx = int(os.environ.get("SK_BATCH", 16)), int(os.environ.get("SK_CTX", 65536))
H, HKV, D = 32, 8, 128
gates = [0.9 - 0.001 * h if h % 4 < 2 else 0.1 + 0.001 * h for h in range(H)]
cfg = sk.EngineConfig(quant_bits=4, budget_tokens=4096, reuse_interval=4, local_blocks=4)
ly = BatchedLayer(cfg, sk.classify_heads(gates, 0.5, 1, 4), B, HKV, D, device="cuda:0", capacity_tokens=ctx + 64)
g = torch.Generator(device="cuda").manual_seed(0)
for b in range(B):
    k = torch.randn((ctx, HKV, D), generator=g, device="cuda", dtype=torch.float16)
    ly.load_context(b, k, k)
dg = DecodeGraph([ly], 16, D, record_ledger=False)
dg.q.normal_()
dg.k.normal_()
dg.v.normal_()
for _ in range(8):
    dg.step()
torch.cuda.synchronize()
print("done", ly.pool.tokens_host[0])
