"""Golden run of the REAL reference at BASELINE cfg1:
one Llama-3-8B attention layer (32 Q / 8 KV heads, D = 128), 8k-token prefill
then 256 decode steps, balanced 50% streaming heads (2 retrieval + 2
streaming per KV group; sink 64 + local 256 tokens), page 64, logical 16,
KV4, budget 4096, reuse 4.

Run in the build container, where the reference is importable (about 70 s):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_cfg1.py

Inputs are NOT stored: they are regenerated bit-identically from
``inputs(seed)`` below (numpy's PCG64 stream; their sha256 is stored and
checked).  Stored: the prefill and decode ledgers, the selector counts,
every step's index tables and invoked flags, the prefill output at 256
sampled rows plus per-head sums over all rows, every decode output
(fp16-rounded), and sha256 digests of every KV head's final pages (codes,
scale/zero, logical-page stats) in the canonical form of ``page_digest``.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "cfg1_ref.npz")

N = S = 8192
H, HKV, D = 32, 8, 128
STEPS = 256
SEED = 2502
SAMPLE_ROWS = np.r_[0:64, 4032:4160, 8128:8192]
CFG = dict(physical_page=64, logical_page=16, quant_bits=4, budget_tokens=4096, reuse_interval=4,
           sink_blocks=1, local_blocks=4, target_sparsity=0.5)


def balanced_gates(h: int = H) -> list:
    """2 retrieval + 2 streaming query heads per KV group."""
    return [0.9 - 0.001 * i if i % 4 < 2 else 0.1 + 0.001 * i for i in range(h)]


def inputs(seed: int = SEED):
    """fp16-valued float32 arrays: prefill q/k/v, then per-step decode rows."""
    rng = np.random.default_rng(seed)
    f = lambda *s: rng.standard_normal(s).astype(np.float16).astype(np.float32)  # noqa: E731
    q, k, v = f(N, H, D), f(S, HKV, D), f(S, HKV, D)
    qn, kn, vn = f(STEPS, H, D), f(STEPS, HKV, D), f(STEPS, HKV, D)
    return q, k, v, qn, kn, vn


def input_digest(arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def page_digest(pages) -> str:
    """Canonical sha256 of a KV head's live pages (reference PhysicalPage fields)."""
    h = hashlib.sha256()
    for p in pages:
        tc = p.token_count
        h.update(np.array([p.page_id, tc], np.int64).tobytes())
        for a in (p.k_codes[:tc], p.v_codes[:tc]):
            h.update(np.ascontiguousarray(np.asarray(a, np.float64)).tobytes())
        for a in (p.k_scale, p.k_zero, p.v_scale, p.v_zero):
            h.update(np.ascontiguousarray(np.asarray(a, np.float64)).tobytes())
        for s in p.stats:
            h.update(np.asarray(s.k_min, np.float64).tobytes())
            h.update(np.asarray(s.k_max, np.float64).tobytes())
            h.update(np.array([s.covered_tokens], np.int64).tobytes())
    return h.hexdigest()


def main() -> None:
    sys.dont_write_bytecode = True
    sys.path.insert(0, os.environ.get("SPARSEKV_REF", "/root/reference/pkg/src"))
    from sparsekv import Engine, EngineConfig, Workload, classify_heads

    q, k, v, qn, kn, vn = inputs()
    cfg = EngineConfig(**CFG)
    profiles = classify_heads(balanced_gates(), cfg.target_sparsity, cfg.sink_blocks, cfg.local_blocks)
    eng = Engine(cfg, profiles)
    t0 = time.perf_counter()
    pre = eng.prefill(Workload(q, k, v))
    t_pre = time.perf_counter() - t0
    ledger_pre = (eng.ledger.visited("prefill"), eng.ledger.total("prefill"))
    width = max(CFG["budget_tokens"] // CFG["physical_page"], 8) + CFG["sink_blocks"] + CFG["local_blocks"]
    tables = np.full((STEPS, H, width), -1, np.int16)
    invoked = np.zeros((STEPS, HKV), np.int8)
    dec = np.zeros((STEPS, H, D), np.float16)
    t0 = time.perf_counter()
    for t in range(STEPS):
        res = eng.decode_step(qn[t], kn[t], vn[t])
        dec[t] = res.output.astype(np.float16)
        for tb in res.index_tables:
            tables[t, tb.head, :len(tb.positions)] = tb.positions
        for kv, ran in res.invoked.items():
            invoked[t, kv] = ran
    t_dec = time.perf_counter() - t0
    digests = np.array([page_digest(eng.cache.pool_of(kv).live_pages()) for kv in range(HKV)])
    tiles = sorted(eng.ledger.tiles.items())
    np.savez_compressed(
        OUT, input_sha256=input_digest([q, k, v, qn, kn, vn]), gates=np.array(balanced_gates()),
        roles=np.array([p.role == "retrieval" for p in profiles], np.int8),
        sample_rows=SAMPLE_ROWS, prefill_rows=pre[SAMPLE_ROWS].astype(np.float32),
        prefill_head_sum=pre.astype(np.float64).sum(axis=(0, 2)),
        prefill_head_sumsq=(pre.astype(np.float64) ** 2).sum(axis=(0, 2)),
        ledger_prefill=np.array(ledger_pre, np.int64),
        ledger_decode=np.array((eng.ledger.visited("decode"), eng.ledger.total("decode")), np.int64),
        tile_keys=np.array([f"{st}:{h}" for (st, h), _ in tiles]),
        tile_vals=np.array([val for _, val in tiles], np.int64),
        selector_calls=np.array([eng.ledger.selector_invocations.get(kv, 0) for kv in range(HKV)], np.int64),
        tables=tables, invoked=invoked, decode_out=dec, page_digests=digests,
        seconds=np.array([t_pre, t_dec]))
    print(f"wrote {OUT}: prefill {t_pre:.1f} s, {STEPS} decode steps {t_dec:.1f} s, ledgers {ledger_pre} / "
          f"{(eng.ledger.visited('decode'), eng.ledger.total('decode'))}, "
          f"selector calls {eng.ledger.total_selector_invocations}")


if __name__ == "__main__":
    main()
