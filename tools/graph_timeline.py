"""Kernel timeline of one replayed decode step (CUPTI via torch.profiler):
cfg4 batched (SK_MODE=batched, default) or cfg2 (SK_MODE=single), 8 layers.
Prints each kernel's start offset, duration and the idle gap before it."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2502_14866_b200 as sk
from paper_2502_14866_b200.batch import BatchedLayer
from paper_2502_14866_b200.decode_graph import DecodeGraph

L = int(os.environ.get("SK_LAYERS", 8))
mode = os.environ.get("SK_MODE", "batched")
B, ctx = (16, 65536) if mode == "batched" else (1, 131072)
H, HKV, D = 32, 8, 128
gates = [0.9 - 0.001 * i if i % 4 < 2 else 0.1 + 0.001 * i for i in range(H)]
prof_ = sk.classify_heads(gates, 0.5, 1, 4)
cfg = sk.EngineConfig(local_blocks=4)
g = torch.Generator(device="cuda").manual_seed(0)
layers = []
for _ in range(L):
    ly = BatchedLayer(cfg, prof_, B, HKV, D, device="cuda:0", capacity_tokens=ctx + 80)
    for b in range(B):
        k = torch.randn((ctx, HKV, D), generator=g, device="cuda", dtype=torch.float16)
        ly.load_context(b, k, k)
    layers.append(ly)
dg = DecodeGraph(layers, 68, D, record_ledger=False)
dg.q.normal_(generator=g)
dg.k.normal_(generator=g)
dg.v.normal_(generator=g)
for _ in range(8):
    dg.step()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
for step_kind in range(4):
    flush.zero_()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        dg.step()
        torch.cuda.synchronize()
    ev = sorted([e for e in p.events() if e.device_type == torch.autograd.DeviceType.CUDA and "elementwise" not in e.name],
                key=lambda e: e.time_range.start)
    if not ev:
        continue
    t0 = ev[0].time_range.start
    print(f"--- step {step_kind}: {len(ev)} kernels, span {(ev[-1].time_range.end - t0):.1f} us")
    last_end = t0
    for e in ev:
        st, en = e.time_range.start, e.time_range.end
        print(f"  {e.name.split('(')[0][-40:]:40s} start {st - t0:8.1f} dur {en - st:7.1f} gap {st - last_end:6.1f}")
        last_end = max(last_end, en)
