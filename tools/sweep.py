"""Measured sweeps over BASELINE.json configs 3 and 5 on one B200 (one layer
each; per-layer numbers scale linearly in layers):

  cfg5  Llama-2-7B MHA shapes (32 Q / 32 KV heads, D=128), context
        32k..192k x streaming-head fraction {0, .25, .5, .75} x budget
        {2048, 4096, 8192}: K4 prefill ms + TFLOP/s, one decode step (K2 +
        K3 + K1, CUDA graph) in us.
  cfg3  Llama-3-8B shapes at 256k context on one GPU (the per-rank work of
        KV-head sharding at g = 1; g > 1 ranks do 8/g KV heads each).

Prints one JSON line per point (and writes them to $SK_SWEEP_OUT if set).
"""
import json
import math
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2502_14866_b200 as sk
from paper_2502_14866_b200.attn import run_prefill
from paper_2502_14866_b200.decode_graph import DecodeGraph

D = 128


def gates_for(h, hkv, frac):
    """`frac` of the heads streaming, spread evenly over KV groups (GQA: the
    same count in every group, like bench.py's balanced layout)."""
    g = h // hkv
    if g > 1:
        n_s = round(frac * g)
        streaming = {i for i in range(h) if i % g >= g - n_s}
    else:
        order = sorted(range(h), key=lambda i: ((i * 37) % h))
        streaming = set(order[:round(frac * h)])
    return [0.1 + 0.001 * i if i in streaming else 0.9 - 0.001 * i for i in range(h)]


def point(h, hkv, ctx, frac, budget, decode_steps=8, reps=3):
    gates = gates_for(h, hkv, frac)
    sparsity = frac if frac > 0 else 0.0
    cfg = sk.EngineConfig(quant_bits=4, budget_tokens=budget, reuse_interval=4, local_blocks=4,
                          target_sparsity=min(sparsity, 0.99))
    prof = [sk.HeadProfile(i, g, sk.STREAMING if g < 0.5 else sk.RETRIEVAL, 1, 4) for i, g in enumerate(gates)]
    eng = sk.Engine(cfg, prof, device="cuda:0", capacity_tokens=ctx + decode_steps + 8)
    gen = torch.Generator(device="cuda").manual_seed(ctx + h)
    q = torch.randn((ctx, h, D), generator=gen, device="cuda", dtype=torch.float16)
    k = torch.randn((ctx, hkv, D), generator=gen, device="cuda", dtype=torch.float16)
    v = torch.randn((ctx, hkv, D), generator=gen, device="cuda", dtype=torch.float16)
    eng.prefill_device(q, k, v, D)
    plan = eng._plan(ctx, ctx)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run_prefill(q, k, v, plan, 1 / math.sqrt(D))
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    pre_ms = statistics.median(ts)
    flop = int(plan.visited.sum()) * 4 * 64 * 64 * D
    del q
    dg = DecodeGraph([eng], decode_steps + 4, D, record_ledger=False)
    dg.q.normal_(generator=gen)
    dg.k.normal_(generator=gen)
    dg.v.normal_(generator=gen)
    for _ in range(4):
        dg.step()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    dts = []
    for _ in range(decode_steps):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dg.step()
        b.record()
        torch.cuda.synchronize()
        dts.append(a.elapsed_time(b) * 1e3)
    return {"q_heads": h, "kv_heads": hkv, "ctx": ctx, "streaming_frac": frac, "budget": budget,
            "prefill_ms_per_layer": round(pre_ms, 3), "prefill_tflops": round(flop / pre_ms / 1e9, 1),
            "prefill_frac_of_1654": round(flop / pre_ms / 1e9 / 1654.2, 3),
            "visited_tiles": int(plan.visited.sum()), "total_tiles": int(plan.total.sum()),
            "decode_us_per_layer_step": round(statistics.mean(dts), 2)}


def main():
    out = open(os.environ["SK_SWEEP_OUT"], "w") if os.environ.get("SK_SWEEP_OUT") else None
    pts = []
    for ctx in (32768, 65536, 131072, 196608):  # cfg5 context sweep at 50% streaming, budget 4096
        pts.append(("cfg5", 32, 32, ctx, 0.5, 4096))
    for frac in (0.0, 0.25, 0.75):  # cfg5 sparsity sweep at 128k
        pts.append(("cfg5", 32, 32, 131072, frac, 4096))
    for budget in (2048, 8192):  # cfg5 budget sweep at 128k
        pts.append(("cfg5", 32, 32, 131072, 0.5, budget))
    pts.append(("cfg3", 32, 8, 262144, 0.5, 4096))  # cfg3 per-rank work at g = 1
    for name, h, hkv, ctx, frac, budget in pts:
        rec = {"config": name, **point(h, hkv, ctx, frac, budget)}
        line = json.dumps(rec)
        print(line, flush=True)
        if out:
            out.write(line + "\n")
            out.flush()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
