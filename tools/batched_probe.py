"""cfg4 batched decode (B sequences x ctx, per-sequence page tables) through
DecodeGraph over SK_LAYERS layers, L2 flushed per step: us per layer-step
(the bench's decode_batched measurement on fewer layers)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2502_14866_b200 as sk
from paper_2502_14866_b200.batch import BatchedLayer
from paper_2502_14866_b200.decode_graph import DecodeGraph

L, B, ctx = int(os.environ.get("SK_LAYERS", 8)), int(os.environ.get("SK_B", 16)), int(os.environ.get("SK_CTX", 65536))
H, HKV, D = 32, 8, 128
gates = [0.9 - 0.001 * i if i % 4 < 2 else 0.1 + 0.001 * i for i in range(H)]
prof = sk.classify_heads(gates, 0.5, 1, 4)
cfg = sk.EngineConfig(local_blocks=4)
g = torch.Generator(device="cuda").manual_seed(0)
layers = []
for _ in range(L):
    ly = BatchedLayer(cfg, prof, B, HKV, D, device="cuda:0", capacity_tokens=ctx + 80)
    for b in range(B):
        k = torch.randn((ctx, HKV, D), generator=g, device="cuda", dtype=torch.float16)
        ly.load_context(b, k, k)
    layers.append(ly)
dg = DecodeGraph(layers, 72, D, record_ledger=False)
dg.q.normal_(generator=g)
dg.k.normal_(generator=g)
dg.v.normal_(generator=g)
for _ in range(4):
    dg.step()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(28):
    flush.zero_()
    torch.cuda.synchronize()
    a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    dg.step()
    b_.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b_) * 1e3)
print(f"batched decode {B} x {ctx}, {L} layers: {statistics.mean(ts):.1f} us/step ({statistics.mean(ts) / L:.2f} us/layer)")
# host-side cost of DecodeGraph.step (bookkeeping after the replay is enqueued)
import time
hs = []
for _ in range(16):
    torch.cuda.synchronize()
    t = time.perf_counter()
    dg.step()
    hs.append((time.perf_counter() - t) * 1e6)
torch.cuda.synchronize()
print(f"host time per step() call: mean {statistics.mean(hs):.0f} us, max {max(hs):.0f} us")
