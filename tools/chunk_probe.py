"""Chunked-prefill cost on one B200 (cfg2 head geometry, one layer): a C-token
chunk continuing an S0-token cached history of KV4 pages.  Times K1b gather,
K4 over the gathered (S0 + C) keys, the paged K4 (history read through the
page table, no gather) and the whole prefill_chunk with CUDA events (median
of 5, L2 flushed before each), prints one JSON line per (S0, C)."""
import json
import math
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2502_14866_b200 as sk
from paper_2502_14866_b200.attn import run_prefill, run_prefill_paged

H, HKV, D = 32, 8, 128


def timed(fn, flush, reps=5):
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    gates = [0.9 - 0.001 * i if i % 4 < 2 else 0.1 + 0.001 * i for i in range(H)]
    prof = sk.classify_heads(gates, 0.5, 1, 4)
    cfg = sk.EngineConfig(quant_bits=4, local_blocks=4)
    for s0, c in ((131072, 8192), (131072, 2048), (131072, 512), (131072, 256), (32768, 4096)):
        eng = sk.Engine(cfg, prof, device="cuda:0", capacity_tokens=s0 + c)
        g = torch.Generator(device="cuda").manual_seed(s0 + c)
        kh = torch.randn((s0, HKV, D), generator=g, device="cuda", dtype=torch.float16)
        vh = torch.randn((s0, HKV, D), generator=g, device="cuda", dtype=torch.float16)
        eng.cache = None
        eng._group_size = H // HKV
        eng._new_cache(HKV, D, s0 + c)
        eng.cache._user_dim = D
        eng.cache.append_all(kh, vh)
        del kh, vh
        q = torch.randn((c, H, D), generator=g, device="cuda", dtype=torch.float16)
        k = torch.randn((c, HKV, D), generator=g, device="cuda", dtype=torch.float16)
        v = torch.randn((c, HKV, D), generator=g, device="cuda", dtype=torch.float16)
        pool = eng.cache.pool
        t_gather = timed(lambda: pool.gather(extra_tokens=c), flush)
        kf, vf = pool.gather(extra_tokens=c)
        kf[s0:], vf[s0:] = k, v
        plan = eng._plan(c, s0 + c)
        t_attn = timed(lambda: run_prefill(q, kf, vf, plan, 1 / math.sqrt(D)), flush)
        flop = int(plan.visited.sum()) * 4 * 64 * 64 * D
        ref_out = run_prefill(q, kf, vf, plan, 1 / math.sqrt(D))
        del kf, vf
        t_paged = timed(lambda: run_prefill_paged(pool, s0, q, k, v, plan, 1 / math.sqrt(D)), flush)
        pg_out = run_prefill_paged(pool, s0, q, k, v, plan, 1 / math.sqrt(D))
        paged_vs_gather = float((pg_out.float() - ref_out.float()).abs().max())
        t_total = timed(lambda: eng.prefill_chunk_device(q, k, v, D), flush, reps=1)
        gbytes = (s0 * HKV * D // 2 * 2 + (s0 // 64) * HKV * 4 * D * 2 + 2 * s0 * HKV * D * 2) / 1e9
        print(json.dumps({"history": s0, "chunk": c, "gather_ms": round(t_gather, 3),
                          "gather_GBps": round(gbytes / t_gather * 1e3, 1), "k4_ms": round(t_attn, 3),
                          "k4_tflops": round(flop / t_attn / 1e9, 1), "k4_paged_ms": round(t_paged, 3),
                          "k4_paged_tflops": round(flop / t_paged / 1e9, 1),
                          "paged_vs_gather_max_abs": paged_vs_gather, "chunk_total_ms": round(t_total, 3)}),
              flush=True)
        del eng, q, k, v
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
