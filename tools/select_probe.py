"""K2 alone: batched (cfg4: 16 sequences x 64k, 128 streams) and one
sequence at 128k (8 streams), median of 20 launches, L2 flushed between."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2502_14866_b200 as sk
from paper_2502_14866_b200.batch import BatchedLayer
from paper_2502_14866_b200.selector import select_streams

H, HKV, D = 32, 8, 128
gates = [0.9 - 0.001 * h if h % 4 < 2 else 0.1 + 0.001 * h for h in range(H)]
cfg = sk.EngineConfig(quant_bits=4, budget_tokens=4096, reuse_interval=4, local_blocks=4)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for B, ctx in ((16, 65536), (1, 131072)):
    ly = BatchedLayer(cfg, sk.classify_heads(gates, 0.5, 1, 4), B, HKV, D, device="cuda:0", capacity_tokens=ctx + 64)
    g = torch.Generator(device="cuda").manual_seed(0)
    for b in range(B):
        k = torch.randn((ctx, HKV, D), generator=g, device="cuda", dtype=torch.float16)
        ly.load_context(b, k, k)
    pool = ly.pool
    n = pool.n_streams
    q = torch.randn((n, 4, D), generator=g, device="cuda", dtype=torch.float16)
    kp = 64
    out = torch.empty((n, kp), dtype=torch.int32, device="cuda")
    cnt = torch.empty(n, dtype=torch.int32, device="cuda")
    ts = []
    for i in range(23):
        flush.zero_()
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        select_streams(pool, q, 4 * D, D, 4, ly._row_mask, kp, out, cnt, max_pages_hint=pool.page_count(0))
        b_.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b_) * 1e3)
    print(f"select B={B} ctx={ctx} streams={n}: {statistics.median(ts):.1f} us", flush=True)
    del ly, pool
    torch.cuda.empty_cache()
