"""Generate the golden fixtures that pin the oracle (and, through it, the
B200 path) to the REAL reference implementation.

Run in the build container, where the reference is importable:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``sparsekv`` from ``/root/reference/pkg/src`` (read-only), runs it
on seeded fp16-valued inputs (cast to float32, the reference's working
precision) and writes compressed ``.npz`` files next to this
script.  Nothing at test time reads ``/root/reference``; the GPU box only
sees these fixtures.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("SPARSEKV_REF", "/root/reference/pkg/src")
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

import sparsekv  # noqa: E402
from sparsekv.cache import HeadPages  # noqa: E402
from sparsekv import (Engine, EngineConfig, HeadProfile,  # noqa: E402
                      Workload, blockwise_attention, classify_heads,
                      quantize_page, select_pages)
from sparsekv.attn import diagonal_tile, full_causal_schedule, query_tile_count  # noqa: E402
from sparsekv.selector import score_pages  # noqa: E402

D = 128


def f16(rng, shape, scale=1.0):
    return (rng.standard_normal(shape) * scale).astype(np.float16)


def pack_tables(tables):
    width = max(len(t.positions) for t in tables)
    arr = np.full((len(tables), width), -1, np.int32)
    for i, t in enumerate(tables):
        arr[i, :len(t.positions)] = t.positions
    return arr


def snapshot(cache, prefix, out):
    """Flatten every live page of both pools (codes, scale/zero, stats)."""
    recs = []
    for pool_name, pool in (("dense", cache.dense_pool), ("streaming", cache.streaming_pool)):
        for kv in sorted(pool):
            for page in pool[kv].live_pages():
                recs.append((pool_name == "dense", kv, page))
    n = len(recs)
    cap = recs[0][2].capacity
    out[prefix + "page_dense"] = np.array([r[0] for r in recs], np.int8)
    out[prefix + "page_kv"] = np.array([r[1] for r in recs], np.int32)
    out[prefix + "page_index"] = np.array([r[2].page_id for r in recs], np.int32)
    out[prefix + "page_tokens"] = np.array([r[2].token_count for r in recs], np.int32)
    codes_dt = recs[0][2].k_codes.dtype
    kc = np.zeros((n, cap, D), codes_dt)
    vc = np.zeros((n, cap, D), codes_dt)
    for i, (_, _, p) in enumerate(recs):
        kc[i, :p.token_count] = p.k_codes[:p.token_count]
        vc[i, :p.token_count] = p.v_codes[:p.token_count]
    if codes_dt == np.float64:  # bits=None: raw fp16-valued inputs, exact in fp16
        kc, vc = kc.astype(np.float16), vc.astype(np.float16)
    out[prefix + "k_codes"], out[prefix + "v_codes"] = kc, vc
    for name in ("k_scale", "k_zero", "v_scale", "v_zero"):
        out[prefix + name] = np.stack([getattr(r[2], name) for r in recs])
    n_log = cap // cache.logical_page
    smin = np.zeros((n, n_log, D), np.float16)
    smax = np.zeros((n, n_log, D), np.float16)
    cov = np.zeros((n, n_log), np.int32)
    for i, (_, _, p) in enumerate(recs):
        for j, s in enumerate(p.stats):
            smin[i, j], smax[i, j], cov[i, j] = s.k_min, s.k_max, s.covered_tokens
    out[prefix + "stats_min"], out[prefix + "stats_max"] = smin, smax
    out[prefix + "stats_covered"] = cov


def engine_case(path, quant_bits, seed):
    rng = np.random.default_rng(seed)
    n = s = 768
    h, h_kv, steps = 4, 2, 12
    # group 0 mixes roles (dense pool, its streaming row reads it), group 1
    # is all-streaming (streaming pool with eviction).
    gates = [0.9, 0.1, 0.05, 0.15]
    cfg = EngineConfig(quant_bits=quant_bits, budget_tokens=384, reuse_interval=4,
                       sink_blocks=1, local_blocks=2, target_sparsity=0.75)
    profiles = classify_heads(gates, cfg.target_sparsity, cfg.sink_blocks, cfg.local_blocks)
    q, k, v = f16(rng, (n, h, D)), f16(rng, (s, h_kv, D)), f16(rng, (s, h_kv, D))
    eng = Engine(cfg, profiles)
    out = {}
    pre = eng.prefill(Workload(q.astype(np.float32), k.astype(np.float32), v.astype(np.float32)))
    out.update(q=q, k=k, v=v, gates=np.array(gates), prefill_out=pre.astype(np.float32),
               roles=np.array([p.role == "retrieval" for p in profiles], np.int8),
               quant_bits=np.int32(0 if quant_bits is None else quant_bits),
               budget=np.int32(cfg.budget_tokens), reuse=np.int32(cfg.reuse_interval),
               sink=np.int32(cfg.sink_blocks), local=np.int32(cfg.local_blocks),
               sparsity=np.float64(cfg.target_sparsity))
    out["prefill_ledger"] = np.array([eng.ledger.tiles[("prefill", hh)] for hh in range(h)], np.int64)
    qn, kn, vn = f16(rng, (steps, h, D)), f16(rng, (steps, h_kv, D)), f16(rng, (steps, h_kv, D))
    outs, tables, invoked = [], [], []
    for t in range(steps):
        res = eng.decode_step(qn[t].astype(np.float32), kn[t].astype(np.float32),
                              vn[t].astype(np.float32))
        outs.append(res.output.astype(np.float32))
        tab = pack_tables(res.index_tables)
        tables.append(tab)
        invoked.append([int(res.invoked.get(kv, -1)) for kv in range(h_kv)])
    width = max(t.shape[1] for t in tables)
    out["decode_tables"] = np.stack([np.pad(t, ((0, 0), (0, width - t.shape[1])), constant_values=-1)
                                     for t in tables])
    out.update(q_new=qn, k_new=kn, v_new=vn, decode_out=np.stack(outs),
               decode_invoked=np.array(invoked, np.int8))
    out["decode_ledger"] = np.array([eng.ledger.tiles[("decode", hh)] for hh in range(h)], np.int64)
    out["selector_calls"] = np.array([eng.ledger.selector_invocations.get(kv, 0)
                                      for kv in range(h_kv)], np.int64)
    snapshot(eng.cache, "final_", out)
    # a snapshot after prefill alone, from a fresh engine (bulk-append path)
    eng2 = Engine(cfg, profiles)
    eng2.load_context(k.astype(np.float32), v.astype(np.float32))
    snapshot(eng2.cache, "load_", out)
    np.savez_compressed(path, **out)


def select_case(path, seed):
    rng = np.random.default_rng(seed)
    out = {}
    cases = [(640, 1, 256), (4096, 2, 1024), (4608, 4, 2048), (2000, 4, 512), (3000, 3, 1000)]
    for i, (s, rows, budget) in enumerate(cases):
        keys = f16(rng, (s, D), scale=rng.uniform(0.5, 3.0))
        head = HeadPages(0, 64, 16, bits=None, with_stats=True)
        head.append(keys.astype(np.float64), np.zeros((s, D)))
        q = f16(rng, (rows, D))
        sel = select_pages(q.astype(np.float64), head.live_pages(), budget, 64)
        sc = score_pages(q.astype(np.float64), head.live_pages())
        out[f"c{i}_keys"], out[f"c{i}_q"] = keys, q
        out[f"c{i}_budget"] = np.int32(budget)
        out[f"c{i}_sel"] = np.array(sel, np.int32)
        out[f"c{i}_scores"] = sc
    # all-tie case (test_selector.py:138-145 style) at a realistic size
    keys = np.zeros((64 * 40, D), np.float16)
    head = HeadPages(0, 64, 16, bits=None, with_stats=True)
    head.append(keys.astype(np.float64), np.zeros_like(keys, dtype=np.float64))
    out["tie_sel"] = np.array(select_pages(np.ones(D), head.live_pages(), 64 * 10, 64), np.int32)
    out["n_cases"] = np.int32(len(cases))
    np.savez_compressed(path, **out)


def quant_case(path, seed):
    rng = np.random.default_rng(seed)
    out = {}
    specs = [(64, 4), (37, 4), (1, 4), (64, 8), (64, 2), (16, 3), (64, 5), (50, 7), (64, 6)]
    for i, (t, bits) in enumerate(specs):
        raw = f16(rng, (t, D), scale=rng.uniform(0.1, 8.0))
        if i == 0:
            raw[:, 5] = np.float16(1.25)  # constant channel -> scale 1
        codes, scale, zero = quantize_page(raw.astype(np.float64), bits)
        out[f"q{i}_raw"], out[f"q{i}_bits"] = raw, np.int32(bits)
        out[f"q{i}_codes"], out[f"q{i}_scale"], out[f"q{i}_zero"] = codes, scale, zero
    out["n_cases"] = np.int32(len(specs))
    np.savez_compressed(path, **out)


def blockwise_case(path, seed):
    """Ragged / misaligned geometry and custom schedules (ledger + outputs)."""
    rng = np.random.default_rng(seed)
    out = {}
    specs = [(100, 160, 4, 2, 64, 64), (200, 200, 2, 1, 64, 64), (130, 330, 2, 1, 64, 64),
             (256, 256, 2, 2, 128, 64), (96, 96, 2, 1, 32, 16)]
    for i, (n, s, h, h_kv, tq, tk) in enumerate(specs):
        q, k, v = f16(rng, (n, h, D)), f16(rng, (s, h_kv, D)), f16(rng, (s, h_kv, D))
        w = Workload(q.astype(np.float32), k.astype(np.float32), v.astype(np.float32))
        sched = {}
        for hh in range(h):
            for qt in range(query_tile_count(n, tq)):
                full = list(full_causal_schedule(qt, tq, tk, n, s))
                if hh % 2 == 1 and len(full) > 2:  # random partial schedule keeping the diagonal
                    keep = sorted(set(rng.choice(full[:-1], size=len(full) // 2, replace=False).tolist())
                                  | {full[-1]})
                    sched[(hh, qt)] = keep
                else:
                    sched[(hh, qt)] = full
        o, led = blockwise_attention(w, sched, tq, tk, "prefill")
        n_qt = query_tile_count(n, tq)
        n_kt = -(-s // tk)
        mask = np.zeros((h, n_qt, n_kt), np.int8)
        for (hh, qt), tl in sched.items():
            mask[hh, qt, tl] = 1
        out[f"b{i}_q"], out[f"b{i}_k"], out[f"b{i}_v"] = q, k, v
        out[f"b{i}_geom"] = np.array([n, s, h, h_kv, tq, tk], np.int32)
        out[f"b{i}_mask"] = mask
        out[f"b{i}_out"] = o.astype(np.float32)
        out[f"b{i}_ledger"] = np.array([led.tiles[("prefill", hh)] for hh in range(h)], np.int64)
        out[f"b{i}_diag"] = np.array([diagonal_tile(qt, tq, tk, n, s) for qt in range(n_qt)], np.int32)
    out["n_cases"] = np.int32(len(specs))
    np.savez_compressed(path, **out)


def main():
    print("reference sparsekv", sparsekv.__version__, "from", REF)
    engine_case(os.path.join(HERE, "engine_kv4.npz"), 4, seed=101)
    engine_case(os.path.join(HERE, "engine_fp16pages.npz"), None, seed=202)
    select_case(os.path.join(HERE, "select.npz"), seed=303)
    quant_case(os.path.join(HERE, "quantize.npz"), seed=404)
    blockwise_case(os.path.join(HERE, "blockwise.npz"), seed=505)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)), "bytes")


if __name__ == "__main__":
    main()
