"""Multi-layer decode step through DecodeGraph (cfg2 heads, 128k context,
SK_LAYERS layers loaded with load_context), L2 flushed between steps, mean
over whole reuse windows -- the bench's decode measurement on fewer layers."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2502_14866_b200 as sk
from paper_2502_14866_b200.decode_graph import DecodeGraph

L, N, H, HKV, D = int(os.environ.get("SK_LAYERS", 8)), 131072, 32, 8, 128
gates = [0.9 - 0.001 * i if i % 4 < 2 else 0.1 + 0.001 * i for i in range(H)]
prof = sk.classify_heads(gates, 0.5, 1, 4)
cfg = sk.EngineConfig(local_blocks=4)
engines = []
g = torch.Generator(device="cuda").manual_seed(0)
for _ in range(L):
    e = sk.Engine(cfg, prof, device="cuda:0", capacity_tokens=N + 64)
    k = torch.randn((N, HKV, D), generator=g, device="cuda", dtype=torch.float16)
    e.load_context(k, k)
    engines.append(e)
if os.environ.get("SK_PROBE_NO_APPEND"):  # ablation: drop the side-stream K1 from the graph
    from paper_2502_14866_b200 import _lib
    _lib.load().sk_append_pages = lambda *a: 0
dg = DecodeGraph(engines, 40, D, record_ledger=False)
dg.q.normal_(generator=g)
dg.k.normal_(generator=g)
dg.v.normal_(generator=g)
for _ in range(4):
    dg.step()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(32):
    flush.zero_()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    dg.step()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
print(f"decode step {L} layers: {statistics.mean(ts):.1f} us ({statistics.mean(ts) / L:.2f} us/layer)")
