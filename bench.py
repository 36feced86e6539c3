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
# CPU reference: the UNMODIFIED sparsekv package (tools/install_reference.sh
# installs it into baseline/_ref, which travels to the GPU box), timed on the
# host cores on bounded samples of the same workload
# ---------------------------------------------------------------------------

PREFILL_DEPTHS = (255, 1023, 2047)  # q-tiles sampled at 1/8, 1/2 and the end of a 128k prefill


def load_reference():
    """import sparsekv from baseline/_ref (None if it was never installed)."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "sparsekv")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    import sparsekv
    return sparsekv


def host_info():
    """CPU model, logical CPUs and the BLAS thread pool the reference's numpy uses."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        model = next((ln.split(":", 1)[1].strip() for ln in out.splitlines() if ln.startswith("Model name")), None)
    except Exception:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        blas = max((p["num_threads"] for p in threadpool_info() if p.get("user_api") == "blas"), default=None)
    except Exception:
        pass
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "blas_threads": blas,
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS")}


def ref_profiles(ref):
    return ref.classify_heads(balanced_gates(), 0.5, SINK, LOCAL)


def ref_visited_per_layer(ref, ctx: int) -> int:
    """Ledger visited tiles of one cfg2 layer by the reference's own schedules (engine.py:152-165)."""
    n_tiles = ctx // PAGE
    prof = ref_profiles(ref)
    lam = sum(len(ref.streaming_schedule(n_tiles, p, qt).tiles()) for p in prof if p.role != "retrieval"
              for qt in range(n_tiles))
    dense = sum(1 for p in prof if p.role == "retrieval") * n_tiles * (n_tiles + 1) // 2
    return lam + dense


def ref_prefill_tile(ref, q_rows, k_hist, v_hist, qt: int):
    """The reference's blockwise_attention on query tile qt of a 128k prefill,
    all heads, as the sliced workload (the tile's 64 query rows over the
    (qt+1)*64-token history; SURVEY 8c item 2 -- rows identical to the full
    prefill's).  Returns (output [64, H, D], seconds, visited tiles)."""
    prof = ref_profiles(ref)
    n_tiles = (qt + 1)
    sched = {(h, 0): (list(range(qt + 1)) if prof[h].role == "retrieval" else
                      ref.streaming_schedule(n_tiles, prof[h], qt).tiles()) for h in range(H)}
    w = ref.Workload(q_rows, k_hist, v_hist)
    t0 = time.perf_counter()
    out, led = ref.blockwise_attention(w, sched, 64, PAGE, stage="prefill")
    return out, time.perf_counter() - t0, led.visited()


def ref_decode_window(ref, k_hist, v_hist, rng, steps: int = REUSE):
    """One reuse window (1 selection + REUSE-1 reuse steps) of the reference
    Engine.decode_step at the full context, after load_context (untimed)."""
    cfg = ref.EngineConfig(physical_page=PAGE, logical_page=LOGICAL, quant_bits=BITS, budget_tokens=BUDGET,
                           reuse_interval=REUSE, sink_blocks=SINK, local_blocks=LOCAL, target_sparsity=0.5)
    eng = ref.Engine(cfg, ref_profiles(ref))
    eng.load_context(k_hist, v_hist)
    f = lambda *sh: rng.standard_normal(sh).astype(np.float16).astype(np.float32)  # noqa: E731
    t0 = time.perf_counter()
    for _ in range(steps):
        eng.decode_step(f(H, D), f(HKV, D), f(HKV, D))
    return (time.perf_counter() - t0) / steps


def ref_cfg1(ref, decode_steps: int = 64):
    """BASELINE cfg1 measured in full (no extrapolation): one layer, 8k
    prefill, then `decode_steps` decode steps (tests/golden/make_cfg1.py
    pins the same run's outputs)."""
    rng = np.random.default_rng(1)
    f = lambda *sh: rng.standard_normal(sh).astype(np.float16).astype(np.float32)  # noqa: E731
    n = 8192
    cfg = ref.EngineConfig(physical_page=PAGE, logical_page=LOGICAL, quant_bits=BITS, budget_tokens=BUDGET,
                           reuse_interval=REUSE, sink_blocks=SINK, local_blocks=LOCAL, target_sparsity=0.5)
    eng = ref.Engine(cfg, ref_profiles(ref))
    w = ref.Workload(f(n, H, D), f(n, HKV, D), f(n, HKV, D))
    t0 = time.perf_counter()
    eng.prefill(w)
    t_pre = time.perf_counter() - t0
    t0 = time.perf_counter()
    for _ in range(decode_steps):
        eng.decode_step(f(H, D), f(HKV, D), f(HKV, D))
    t_dec = (time.perf_counter() - t0) / decode_steps
    return {"prefill_ms": round(t_pre * 1e3, 1), "decode_us_per_step": round(t_dec * 1e6, 1),
            "decode_steps": decode_steps, "ctx": n, "layers": 1}


def parity_line(out, ref_out) -> dict:
    o = np.asarray(out, np.float64)
    r = np.asarray(ref_out, np.float64)
    err = float(np.abs(o - r).max())
    ot, rt = o.transpose(1, 0, 2).reshape(o.shape[1], -1), r.transpose(1, 0, 2).reshape(r.shape[1], -1)
    cos = (ot * rt).sum(1) / (np.linalg.norm(ot, axis=1) * np.linalg.norm(rt, axis=1) + 1e-30)
    return {"max_abs": err, "min_cos": float(cos.min())}


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
    from paper_2502_14866_b200.sharding import shard_heads, shard_profiles
    shard = shard_heads(H, HKV, rank, world)  # KV-head block partition
    hkv, h = shard.num_kv_heads, shard.num_heads
    gates = balanced_gates()
    prof_all = sk.classify_heads(gates, 0.5, SINK, LOCAL)
    prof = shard_profiles(prof_all, shard)
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
    if world > 1:  # two head-major gather buffers: layer l's all-gather overlaps layer l+1's attention
        gather = [torch.empty((world, ctx, h, D), dtype=torch.float16, device=dev) for _ in range(2)]

    def prefill_step():
        pending = [None, None]
        for layer in range(L):
            out = engines[layer].prefill_device(qs[layer], ks[layer], vs[layer], D)
            if world > 1:
                if pending[layer % 2] is not None:
                    pending[layer % 2].wait()
                pending[layer % 2] = dist.all_gather_into_tensor(gather[layer % 2], out, async_op=True)
        for w in pending:
            if w is not None:
                w.wait()

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
    # layer 0's output and inputs at the sampled q-tiles, for the reference check below
    sample = None
    if rank == 0 and world == 1 and not args.no_cpu and load_reference() is not None \
            and ctx >= 64 * (max(PREFILL_DEPTHS) + 1):
        out0 = engines[0].prefill_device(qs[0], ks[0], vs[0], D)
        r1 = 64 * (max(PREFILL_DEPTHS) + 1)
        sample = {"gpu": {qt: out0[64 * qt:64 * qt + 64].float().cpu().numpy() for qt in PREFILL_DEPTHS},
                  "q": {qt: qs[0][64 * qt:64 * qt + 64].float().cpu().numpy() for qt in PREFILL_DEPTHS},
                  "k": ks[0][:r1].float().cpu().numpy(), "v": vs[0][:r1].float().cpu().numpy()}
        del out0
    hbm_peak, tf_peak, peak_kind = peaks()
    achieved_tf = flop_layer / (k4_ms * 1e-3) / 1e12

    # ---- decode: CUDA-graph replay of the 32-layer step ----------------------
    dg = DecodeGraph(engines, dec_steps + 4, D, record_ledger=False, group=dist.group.WORLD if world > 1 else None)
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
        dg.step()  # world > 1: one all-gather of head outputs per layer, inside the graph
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
        bdg = DecodeGraph(blayers, dec_steps + 4, D, record_ledger=False,
                          group=dist.group.WORLD if world > 1 else None)
        bq = [(torch.randn((L, B * h, D), generator=gq, device=dev, dtype=torch.float16),
               torch.randn((L, B * hkv, D), generator=gq, device=dev, dtype=torch.float16),
               torch.randn((L, B * hkv, D), generator=gq, device=dev, dtype=torch.float16)) for _ in range(4)]
        for i in range(4):
            bdg.q.copy_(bq[i][0]); bdg.k.copy_(bq[i][1]); bdg.v.copy_(bq[i][2])  # noqa: E702
            bdg.step()
        bts = []
        with Clocks(local_rank) as bclk:
            for i in range(n_dec):
                flush.zero_()
                torch.cuda.synchronize()
                bdg.q.copy_(bq[i % 4][0]); bdg.k.copy_(bq[i % 4][1]); bdg.v.copy_(bq[i % 4][2])  # noqa: E702
                if world > 1:
                    dist.barrier()
                a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                bdg.step()
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

    # ---- the reference (baseline/_ref) on layer 0's own inputs: parity of the
    #      sampled 128k q-tiles, and the cpu_baseline timing of the same work ----
    cpu, parity = None, None
    if sample is not None:
        cpu, parity = reference_against_gpu(load_reference(), sample, ctx, L)
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
        res["cpu_baseline"] = cpu
    if parity is not None:
        res["parity"] = parity
    if args.cfg1:
        res["cfg1"] = run_cfg1_gpu(sk, cfg, prof_all, dev)
    return res


def reference_against_gpu(ref, sample, ctx: int, layers: int):
    """Run the reference on layer 0's sampled q-tiles (the GPU's own inputs):
    per-tile parity of the 128k prefill, and the CPU timing extrapolated by
    the reference's visited-tile count; plus one decode reuse window at 128k."""
    t_pre, vis = 0.0, 0
    par = {}
    for qt in PREFILL_DEPTHS:
        r1 = 64 * (qt + 1)
        out, t, v = ref_prefill_tile(ref, sample["q"][qt], sample["k"][:r1], sample["v"][:r1], qt)
        t_pre += t
        vis += v
        par[str(qt)] = parity_line(sample["gpu"][qt], out)
    per_layer = ref_visited_per_layer(ref, ctx)
    t_dec = ref_decode_window(ref, sample["k"], sample["v"], np.random.default_rng(3))
    info = host_info()
    cpu = {"value": round(t_pre / vis * per_layer * layers * 1e3, 1), "unit": "ms",
           "cores": info["blas_threads"] or 1, "kind": "reference",
           "sample": (f"unmodified sparsekv (baseline/_ref) blockwise_attention on layer 0's own q-tiles "
                      f"{list(PREFILL_DEPTHS)} x {H} heads of the 128k prefill ({vis} visited 64x64 tiles, "
                      f"{t_pre:.1f} s), extrapolated by the reference's visited-tile count ({per_layer}/layer) "
                      f"to {layers} layers; decode: Engine.load_context(128k) + one reuse window "
                      f"({REUSE} steps) of one layer, x{layers} layers"),
           "decode_us_per_step": round(t_dec * layers * 1e6, 1), "host": info}
    worst = {"max_abs": max(p["max_abs"] for p in par.values()), "min_cos": min(p["min_cos"] for p in par.values())}
    parity = {"prefill_sampled_tiles_vs_reference": par, "worst": worst, "tolerance": {"max_abs": 2e-2, "min_cos": 0.9999},
              "ok": worst["max_abs"] <= 2e-2 and worst["min_cos"] >= 0.9999,
              "what": "layer 0 of the timed 128k prefill: q-tiles vs sparsekv.blockwise_attention on the same inputs"}
    return cpu, parity


def run_cfg1_gpu(sk, cfg, prof, dev):
    """BASELINE cfg1 on the GPU, for the measured-vs-measured comparison with
    the reference's full cfg1 run: one layer, 8k prefill (ms) and the decode
    step (us, CUDA graph, selection every 4th step)."""
    import torch

    from paper_2502_14866_b200.decode_graph import DecodeGraph
    n = 8192
    g = torch.Generator(device=dev).manual_seed(8)
    q, k, v = (torch.randn((n, hh, D), generator=g, device=dev, dtype=torch.float16) for hh in (H, HKV, HKV))
    eng = sk.Engine(cfg, prof, device=dev, capacity_tokens=n + 80)
    ts = []
    for i in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        eng.prefill_device(q, k, v, D)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    dg = DecodeGraph([eng], 72, D, record_ledger=False)
    for i in range(4):
        dg.step()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for i in range(64):
        dg.step()
    b.record()
    torch.cuda.synchronize()
    return {"prefill_ms": round(statistics.median(ts[3:]), 3), "decode_us_per_step": round(a.elapsed_time(b) / 64 * 1e3, 2),
            "ctx": n, "layers": 1, "what": "cfg1 (1 layer, 8k, 32/8/128, balanced, KV4, budget 4096, reuse 4); warm L2"}


def run_reference(args, rank, world):
    """The reference arm: the UNMODIFIED sparsekv (baseline/_ref, its public
    API and stock numpy code path) on the host cores, rank 0 only.  Each step
    is one 64-row query tile (all heads) of the cfg2 128k prefill, cycling
    through PREFILL_DEPTHS; `value` extrapolates the measured cost per visited
    tile to the 32-layer prefill by the reference's own visited-tile count.
    Also measured, not extrapolated: one decode reuse window at 128k, and
    BASELINE cfg1 in full (8k prefill + 64 decode steps)."""
    if rank != 0:
        return None
    ref = load_reference()
    if ref is None:
        return {"impl": "reference", "unavailable": "sparsekv not installed in baseline/_ref (tools/install_reference.sh)"}
    t_start = time.perf_counter()
    rng = np.random.default_rng(args.seed)
    f = lambda *sh: rng.standard_normal(sh).astype(np.float16).astype(np.float32)  # noqa: E731
    ctx = args.ctx
    r1 = min(ctx, 64 * (max(PREFILL_DEPTHS) + 1))
    k, v = f(r1, HKV, D), f(r1, HKV, D)
    depths = [qt for qt in PREFILL_DEPTHS if 64 * (qt + 1) <= ctx]
    per_layer = ref_visited_per_layer(ref, ctx)
    for i in range(args.warmup):
        qt = depths[i % len(depths)]
        ref_prefill_tile(ref, f(64, H, D), k[:64 * (qt + 1)], v[:64 * (qt + 1)], qt)
    t_tot, vis_tot, step_ms = 0.0, 0, []
    for i in range(args.steps):
        qt = depths[i % len(depths)]
        _, t, vis = ref_prefill_tile(ref, f(64, H, D), k[:64 * (qt + 1)], v[:64 * (qt + 1)], qt)
        t_tot += t
        vis_tot += vis
        step_ms.append(t / vis * per_layer * args.layers * 1e3)
    val = t_tot / vis_tot * per_layer * args.layers * 1e3
    t_dec = ref_decode_window(ref, k, v, rng)
    cfg1 = ref_cfg1(ref)
    info = host_info()
    cpu = {"value": round(val, 1), "unit": "ms", "cores": info["blas_threads"] or 1, "kind": "reference",
           "sample": (f"{args.steps} timed steps, each one 64-row query tile x {H} heads of the 128k prefill "
                      f"(depths {depths} in turn; {vis_tot} visited tiles, {t_tot:.1f} s), extrapolated by "
                      f"the reference's visited-tile count ({per_layer}/layer) to {args.layers} layers"),
           "host": info}
    return {"metric": METRIC, "impl": "reference", "value": round(val, 1), "unit": "ms", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(val, 1), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic N(0,1) fp16-valued, seeded",
            "config": {"workload": "cfg2 (as our arm): Llama-3-8B attention shapes x 32 layers, 128k prefill + decode, "
                                   "balanced 50% streaming, KV4, budget 4096, reuse 4 -- sampled and extrapolated",
                       "layers": args.layers, "ctx": ctx},
            "cpu_baseline": cpu,
            "step_ms_extrapolated": [round(x, 1) for x in step_ms],
            "decode": {"us_per_step": round(t_dec * args.layers * 1e6, 1),
                       "what": "Engine.decode_step at 128k, one reuse window, x32 layers (measured per layer)"},
            "cfg1_measured": cfg1,
            "e2e": {"value": round(val, 1), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": round(time.perf_counter() - t_start, 1)}


def plan_only(rank: int, world: int):
    """The rank launch and KV-head partition of the multi-GPU bench, without
    GPU work: every rank derives its shard (sharding.shard_heads), the shards
    are all-gathered over gloo, and rank 0 checks they tile all heads."""
    import torch
    import torch.distributed as dist

    from paper_2502_14866_b200.sharding import shard_heads
    if world > 1:
        dist.init_process_group("gloo")
    sh = shard_heads(H, HKV, rank, world)
    mine = torch.tensor([sh.q_begin, sh.q_end, sh.kv_begin, sh.kv_end])
    allp = [torch.zeros_like(mine) for _ in range(world)]
    if world > 1:
        dist.all_gather(allp, mine)
        dist.destroy_process_group()
    else:
        allp = [mine]
    if rank != 0:
        return None
    qs = [h for a, b, _, _ in (t.tolist() for t in allp) for h in range(a, b)]
    ks = [h for _, _, a, b in (t.tolist() for t in allp) for h in range(a, b)]
    return {"plan_only": True, "world": world, "shards": [t.tolist() for t in allp],
            "covers_all_heads": qs == list(range(H)) and ks == list(range(HKV))}


def _free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` run without torchrun: re-launch this script under
    torch.distributed.run with N ranks (one per GPU) on 127.0.0.1."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


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
    ap.add_argument("--plan-only", action="store_true",
                    help="launch the ranks and check the KV-head shard plan over gloo (no GPU work)")
    ap.add_argument("--no-cfg1", dest="cfg1", action="store_false", help="skip the cfg1 (8k) GPU timing")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.plan_only:
        res = plan_only(rank, world)
    elif args.impl == "reference":
        res = run_reference(args, rank, world)
    else:
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(local_rank)
            # NCCL INIT lines (rank count, NVLS) on stderr; stdout stays the one JSON line
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
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
