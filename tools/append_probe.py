"""K1 bulk append (sk_append_pages via DevicePool.append): one 128k-token
KV4 context of 8 KV heads, timed with CUDA events; prints GB/s of the
algorithmic traffic (raw K/V read + codes, bounds and key stats written)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2502_14866_b200 as sk

N, HKV, D, H = 131072, 8, 128, 32
gates = [0.9 - 0.001 * i if i % 4 < 2 else 0.1 + 0.001 * i for i in range(H)]
prof = sk.classify_heads(gates, 0.5, 1, 4)
g = torch.Generator(device="cuda").manual_seed(0)
k = torch.randn((N, HKV, D), generator=g, device="cuda", dtype=torch.float16)
v = torch.randn((N, HKV, D), generator=g, device="cuda", dtype=torch.float16)
ts = []
for it in range(12):
    e = sk.Engine(sk.EngineConfig(quant_bits=4), prof, device="cuda:0", capacity_tokens=N + 64)
    e.load_context(k[:64], v[:64])  # allocate the pool (one page), then time the bulk append
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    e.cache.append_all(k[64:], v[64:])
    b.record()
    torch.cuda.synchronize()
    if it >= 2:
        ts.append(a.elapsed_time(b) * 1e3)
    del e
pages = (N - 64) // 64 * HKV
dense = HKV  # stats for dense streams only (approx: all heads counted)
bytes_ = (N - 64) * HKV * D * 2 * 2 + pages * (64 * D + 8 * D) + pages * 4 * 2 * D * 2
t = statistics.median(ts)
print(f"bulk append {N - 64} tokens x {HKV} streams: {t:.1f} us, {bytes_ / t / 1e3:.0f} GB/s (upper-bound bytes)")
