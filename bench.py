"""Benchmark: LServe sparse-attention prefill + decode at 128k context,
Llama-3-8B attention shapes (BASELINE.json cfg2), on 1..8 B200s.

One JSON line (rank 0).  `value` = prefill wall time of all 32 layers at
128k context (device-resident inputs, CUDA events, max over ranks); the
decode step (32 layers, CUDA-graph replay, selection every 4th step) is
reported in `decode`.  Multi-GPU: KV heads are sharded (strong scaling),
one NCCL all-gather of head outputs per layer.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Sparse-attn prefill ms & decode µs/step at 128k ctx (Llama-3-8B shapes)"
H, HKV, D = 32, 8, 128
PAGE, LOGICAL, BUDGET, REUSE, SINK, LOCAL, BITS = 64, 16, 4096, 4, 1, 4, 4


def balanced_gates(n=H):
    """2 retrieval + 2 streaming query heads per KV group."""
    return [0.9 - 0.001 * h if h % 4 < 2 else 0.1 + 0.001 * h for h in range(n)]


def ncu_traffic(kernel):
    """dram read+write bytes per launch of `kernel` from the newest committed
    ncu --set full capture (profiles/rNN_ncu_traffic.json), else None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_traffic.json")))
    if not files:
        return None
    rec = json.load(open(files[-1]))["kernels"].get(kernel)
    return None if rec is None else int(rec["dram_read_bytes"] + rec["dram_write_bytes"])


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self._stop = gpu, [], threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and "Active" in r[5 + i]
                          and "Not" not in r[5 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU reference (oracle port) on a bounded sample
# ---------------------------------------------------------------------------


def cpu_reference_sample(ctx: int, layers: int, seed: int = 0, budget_s: float = 20.0):
    """Time the reference algorithm (oracle port, numpy) on a bounded sample
    of the same workload and extrapolate to the metric.  Returns dict."""
    from oracle import sparsekv_oracle as O

    threads = os.environ.get("OPENBLAS_NUM_THREADS") or str(os.cpu_count())
    rng = np.random.default_rng(seed)
    roles = O.assign_roles(balanced_gates(), 0.5, SINK, LOCAL)
    n_tiles = ctx // 64
    # prefill sample: whole query tiles (all 32 heads) at a few depths
    qts = [q for q in (255, 1023, 2047) if q < n_tiles]
    vis_sample = 0
    t_pre = 0.0
    for qt in qts:
        if t_pre > budget_s * 0.6:
            break
        r1 = (qt + 1) * 64
        q = rng.standard_normal((64, H, D)).astype(np.float16).astype(np.float32)
        k = rng.standard_normal((r1, HKV, D)).astype(np.float16).astype(np.float32)
        v = rng.standard_normal((r1, HKV, D)).astype(np.float16).astype(np.float32)
        sched = {(h, 0): (list(range(qt + 1)) if roles[h].role == O.RETRIEVAL else
                          O.lambda_tiles(n_tiles, SINK, LOCAL, qt)) for h in range(H)}
        t0 = time.perf_counter()
        O.tiled_attention(q, k, v, sched, 64, 64, O.PREFILL)
        t_pre += time.perf_counter() - t0
        vis_sample += sum(len(t) for t in sched.values())
    vis_layer = sum((qt + 1) if roles[h].role == O.RETRIEVAL else len(O.lambda_tiles(n_tiles, SINK, LOCAL, qt))
                    for h in range(H) for qt in range(n_tiles))
    prefill_ms = t_pre / vis_sample * vis_layer * layers * 1e3
    # decode sample: one layer at the full context, one reuse window of steps
    s_dec = ctx
    eng = O.OracleEngine(O.Config(quant_bits=BITS, budget_tokens=BUDGET, reuse_interval=REUSE, sink_blocks=SINK,
                                  local_blocks=LOCAL), roles)
    k = rng.standard_normal((s_dec, HKV, D)).astype(np.float16).astype(np.float32)
    eng.load_context(k, k)
    t0 = time.perf_counter()
    steps = 4
    for _ in range(steps):
        qn = rng.standard_normal((H, D)).astype(np.float32)
        kn = rng.standard_normal((HKV, D)).astype(np.float32)
        eng.decode_step(qn, kn, kn)
    t_dec = (time.perf_counter() - t0) / steps
    dec_step_ms = t_dec * layers * 1e3
    return {"prefill_ms": prefill_ms, "decode_us_per_step": dec_step_ms * 1e3, "cores": int(threads),
            "sample": (f"oracle port (numpy) prefill of query tiles {qts} x 32 heads of one 128k layer "
                       f"({vis_sample} visited 64x64 tiles, {t_pre:.1f}s), extrapolated by visited tiles to "
                       f"{layers} layers; decode: one reuse window ({steps} steps, 1 selection) of one layer at {s_dec} "
                       f"tokens, x{layers} layers"),
            "seconds": t_pre + t_dec * steps}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2502_14866_b200 as sk
    from paper_2502_14866_b200 import _lib
    from paper_2502_14866_b200.attn import run_prefill
    from paper_2502_14866_b200.decode_graph import DecodeGraph

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    _lib.load()
    hkv = HKV // world
    h = H // world
    heads = list(range(rank * h, (rank + 1) * h))
    gates = balanced_gates()
    prof_all = sk.classify_heads(gates, 0.5, SINK, LOCAL)
    prof = [sk.HeadProfile(i, p.gate, p.role, p.sink_blocks, p.local_blocks)
            for i, p in enumerate(prof_all[heads[0]:heads[-1] + 1])]
    cfg = sk.EngineConfig(physical_page=PAGE, logical_page=LOGICAL, quant_bits=BITS, budget_tokens=BUDGET,
                          reuse_interval=REUSE, sink_blocks=SINK, local_blocks=LOCAL, target_sparsity=0.5)
    ctx, L = args.ctx, args.layers
    dec_steps = args.decode_steps
    qs, ks, vs = [], [], []
    for layer in range(L):
        g = torch.Generator(device=dev).manual_seed(1000 * layer + args.seed + 17 * rank)
        qs.append(torch.randn((ctx, h, D), generator=g, device=dev, dtype=torch.float16))
        ks.append(torch.randn((ctx, hkv, D), generator=g, device=dev, dtype=torch.float16))
        vs.append(torch.randn((ctx, hkv, D), generator=g, device=dev, dtype=torch.float16))
    engines = [sk.Engine(cfg, prof, device=dev, capacity_tokens=ctx + dec_steps + 8) for _ in range(L)]
    gather = None
    if world > 1:
        gather = torch.empty((world, ctx, h, D), dtype=torch.float16, device=dev)

    def prefill_step():
        for layer in range(L):
            out = engines[layer].prefill_device(qs[layer], ks[layer], vs[layer], D)
            if world > 1:
                dist.all_gather_into_tensor(gather, out)

    def timed(fn, reps):
        ts = []
        for _ in range(reps):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return ts

    for _ in range(args.warmup):
        timed(prefill_step, 1)
    clk = Clocks(local_rank)
    clk.__enter__()
    pre_ts = timed(prefill_step, args.steps)
    pre_ms = statistics.mean(pre_ts)
    if world > 1:
        t = torch.tensor([pre_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        pre_ms = float(t.item())

    # dominant kernel (K4) alone: events on the launching stream, per layer
    plan = engines[0]._plan(ctx, ctx)
    flop_layer = int(plan.visited.sum()) * 4 * 64 * 64 * D
    k4 = []
    for layer in range(min(L, 8)):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        run_prefill(qs[layer], ks[layer], vs[layer], plan, 1.0 / math.sqrt(D))
        b.record()
        torch.cuda.synchronize()
        k4.append(a.elapsed_time(b))
    k4_ms = statistics.mean(k4)
    hbm_peak, tf_peak, peak_kind = peaks()
    achieved_tf = flop_layer / (k4_ms * 1e-3) / 1e12

    # ---- decode: CUDA-graph replay of the 32-layer step ----------------------
    dg = DecodeGraph(engines, dec_steps + 4, D, record_ledger=False)
    gq = torch.Generator(device=dev).manual_seed(99 + rank)
    step_inputs = [(torch.randn((L, h, D), generator=gq, device=dev, dtype=torch.float16),
                    torch.randn((L, hkv, D), generator=gq, device=dev, dtype=torch.float16),
                    torch.randn((L, hkv, D), generator=gq, device=dev, dtype=torch.float16)) for _ in range(4)]
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def dec_once(i):
        qn, kn, vn = step_inputs[i % 4]
        dg.q.copy_(qn)
        dg.k.copy_(kn)
        dg.v.copy_(vn)
        dg.step()

    for i in range(4):  # warm: one full reuse window
        dec_once(i)
    dec_ts = []
    n_dec = (dec_steps // REUSE) * REUSE
    dec_gather = torch.empty((world,) + tuple(dg.out.shape), dtype=dg.out.dtype, device=dev) if world > 1 else None
    for i in range(n_dec):
        flush.zero_()  # L2 flush between timed steps
        torch.cuda.synchronize()
        qn, kn, vn = step_inputs[i % 4]
        dg.q.copy_(qn)
        dg.k.copy_(kn)
        dg.v.copy_(vn)
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out_l = dg.step()
        if world > 1:  # head outputs of every layer gathered over NVLink (one collective per step)
            dist.all_gather_into_tensor(dec_gather, out_l)
        b.record()
        torch.cuda.synchronize()
        dec_ts.append(a.elapsed_time(b))
    clk.__exit__()
    dec_us = statistics.mean(dec_ts) * 1e3
    if world > 1:
        t = torch.tensor([dec_us], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dec_us = float(t.item())
    n_pages = -(-(ctx + 4 + n_dec) // PAGE)
    k_pages = BUDGET // PAGE
    slot = 9216
    # bytes one decode step must read per layer: union of pages per KV head
    # (selection + 2 extra local pages) + stats of every logical page / reuse
    dec_bytes_layer = hkv * ((k_pages + 2) * slot + (n_pages * 4 * 2 * D * 2) / REUSE)
    dec_gbs = dec_bytes_layer * L * world / (dec_us * 1e-6) / 1e9  # whole job: every rank's KV heads

    # ---- e2e through the public API with host (pinned) buffers ----------------
    e2e_ms = None
    h2d = d2h = 0
    if not args.no_e2e:
        qh = torch.empty((ctx, h, D), dtype=torch.float16).pin_memory()
        kh = torch.empty((ctx, hkv, D), dtype=torch.float16).pin_memory()
        vh = torch.empty((ctx, hkv, D), dtype=torch.float16).pin_memory()
        oh = torch.empty((ctx, h, D), dtype=torch.float16).pin_memory()
        qh.copy_(qs[0].cpu())
        kh.copy_(ks[0].cpu())
        vh.copy_(vs[0].cpu())

        def e2e_step():  # public multi-layer host API: uploads/downloads overlap the kernels
            sk.prefill_layers(engines, [(qh, kh, vh)] * L, [oh] * L)

        timed(e2e_step, 1)
        e2e_ms = statistics.mean(timed(e2e_step, 1))
        h2d = L * (qh.numel() + kh.numel() + vh.numel()) * 2 * world  # whole job: every rank's heads
        d2h = L * oh.numel() * 2 * world

    # ---- cfg4: batched decode, B sequences x batch_ctx tokens, all layers -------
    batched = None
    if args.batch > 0:
        from paper_2502_14866_b200.batch import BatchedLayer

        del qs, ks, vs, engines, dg
        torch.cuda.empty_cache()
        B, bctx = args.batch, args.batch_ctx
        blayers = [BatchedLayer(cfg, prof, B, hkv, D, device=dev, capacity_tokens=bctx + dec_steps + 8)
                   for _ in range(L)]
        for li, ly in enumerate(blayers):
            g = torch.Generator(device=dev).manual_seed(5000 + 100 * li + args.seed + 17 * rank)
            for b in range(B):
                kb = torch.randn((bctx, hkv, D), generator=g, device=dev, dtype=torch.float16)
                vb = torch.randn((bctx, hkv, D), generator=g, device=dev, dtype=torch.float16)
                ly.load_context(b, kb, vb)
            del kb, vb
        bdg = DecodeGraph(blayers, dec_steps + 4, D, record_ledger=False)
        bq = [(torch.randn((L, B * h, D), generator=gq, device=dev, dtype=torch.float16),
               torch.randn((L, B * hkv, D), generator=gq, device=dev, dtype=torch.float16),
               torch.randn((L, B * hkv, D), generator=gq, device=dev, dtype=torch.float16)) for _ in range(4)]
        for i in range(4):
            bdg.q.copy_(bq[i][0]); bdg.k.copy_(bq[i][1]); bdg.v.copy_(bq[i][2])  # noqa: E702
            bdg.step()
        bts = []
        b_gather = torch.empty((world,) + tuple(bdg.out.shape), dtype=bdg.out.dtype, device=dev) if world > 1 else None
        with Clocks(local_rank) as bclk:
            for i in range(n_dec):
                flush.zero_()
                torch.cuda.synchronize()
                bdg.q.copy_(bq[i % 4][0]); bdg.k.copy_(bq[i % 4][1]); bdg.v.copy_(bq[i % 4][2])  # noqa: E702
                if world > 1:
                    dist.barrier()
                a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                bout = bdg.step()
                if world > 1:
                    dist.all_gather_into_tensor(b_gather, bout)
                b_.record()
                torch.cuda.synchronize()
                bts.append(a.elapsed_time(b_))
        b_us = statistics.mean(bts) * 1e3
        if world > 1:
            t = torch.tensor([b_us], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            b_us = float(t.item())
        bn_pages = -(-(bctx + 4 + n_dec) // PAGE)
        b_bytes = L * B * hkv * ((k_pages + 2) * slot + (bn_pages * 4 * 2 * D * 2) / REUSE)
        b_gbs = b_bytes * world / (b_us * 1e-6) / 1e9
        batched = {"config": f"cfg4: {B} sequences x {bctx} tokens, per-sequence page tables, {L} layers, "
                             f"KV4, budget {BUDGET}, reuse {REUSE}", "batch": B, "ctx": bctx,
                   "us_per_step": round(b_us, 2), "steps": n_dec, "clocks": bclk.summary(),
                   "roofline": {"bound": "hbm", "achieved": round(b_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                                "frac": round(b_gbs / hbm_peak, 4), "peak_kind": peak_kind,
                                "bytes_per_step": int(b_bytes * world),
                                "bytes_def": "per layer per sequence: KV heads x (K+2 pages x 9216 B) + stats / reuse"}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_reference_sample(ctx, L)
    res = {
        "metric": METRIC, "value": round(pre_ms, 3), "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(pre_ms, 3), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f16", "data": "synthetic N(0,1) fp16 q/k/v per layer, seeded",
        "config": {"workload": f"cfg2: Llama-3-8B attention shapes x {L} layers, {ctx}-token prefill + decode, "
                               f"balanced 50% streaming heads (sink {SINK * PAGE} + local {LOCAL * PAGE} tokens), "
                               f"page {PAGE}, logical {LOGICAL}, KV{BITS}, budget {BUDGET}, reuse {REUSE}",
                   "layers": L, "ctx": ctx, "q_heads": H, "kv_heads": HKV, "head_dim": D,
                   "parallelism": f"kv-head shard x{world}" if world > 1 else "single GPU",
                   "l2": "inputs 1.6 GB/layer > 126 MB L2 (prefill); 256 MB L2 flush between decode steps"},
        "roofline": {"bound": "tensor", "kernel": "prefill_kernel (K4, tcgen05)", "achieved": round(achieved_tf, 1),
                     "peak": tf_peak, "unit": "TFLOP/s", "frac": round(achieved_tf / tf_peak, 4),
                     "traffic": ncu_traffic("prefill_kernel"), "peak_kind": peak_kind,
                     "flop_per_launch": flop_layer, "launch_ms": round(k4_ms, 3),
                     "flop_def": "ledger visited 64x64 tiles x 4*64*64*D (QK^T + PV)"},
        "decode": {"us_per_step": round(dec_us, 2), "steps": n_dec, "layers": L,
                   "roofline": {"bound": "hbm", "achieved": round(dec_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                                "frac": round(dec_gbs / hbm_peak, 4), "peak_kind": peak_kind,
                                "traffic_decode_kernel": ncu_traffic("decode_kernel"),
                                "traffic_select_kernel": ncu_traffic("select_kernel"),
                                "bytes_per_step": int(dec_bytes_layer * L * world),
                                "bytes_def": "per layer: KV heads x (K+2 pages x 9216 B) + stats (n_logical x 512 B) / reuse"}},
        "e2e": {"value": round(e2e_ms, 3) if e2e_ms else None, "unit": "ms", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "path": "sk.prefill_layers(engines, pinned host q/k/v per layer, pinned host outputs): per-layer Engine.prefill_device with the H2D of layer l+1 and the D2H of layer l-1 overlapping layer l"},
        "decode_batched": batched,
        "gpu_launches": L * 3 + L * (1 if world > 1 else 0),
        "clocks": clk.summary(),
    }
    if cpu is not None:
        res["cpu_baseline"] = {"value": round(cpu["prefill_ms"], 1), "unit": "ms", "cores": cpu["cores"],
                               "kind": "port", "sample": cpu["sample"],
                               "decode_us_per_step": round(cpu["decode_us_per_step"], 1)}
    return res


def run_reference(args, rank, world):
    if rank != 0:
        return None
    t0 = time.perf_counter()
    cpu = cpu_reference_sample(args.ctx, args.layers)
    val = cpu["prefill_ms"]
    return {"metric": METRIC, "impl": "reference", "value": round(val, 1), "unit": "ms", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(val, 1), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic N(0,1) fp16-valued, seeded",
            "config": {"workload": "cfg2 (same as ours), oracle port on host cores, bounded sample",
                       "layers": args.layers, "ctx": args.ctx},
            "cpu_baseline": {"value": round(val, 1), "unit": "ms", "cores": cpu["cores"], "kind": "port",
                             "sample": cpu["sample"]},
            "decode": {"us_per_step": round(cpu["decode_us_per_step"], 1)},
            "e2e": {"value": round(val, 1), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": round(time.perf_counter() - t0, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--ctx", type=int, default=131072)
    ap.add_argument("--decode-steps", type=int, default=64)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--batch", type=int, default=16, help="cfg4 batched decode sequences (0 = skip)")
    ap.add_argument("--batch-ctx", type=int, default=65536)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        res = run_reference(args, rank, world)
    else:
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        res = run_ours(args, rank, world, local_rank)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
