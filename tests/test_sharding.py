"""KV-head sharding on CPU: world_size-2 ``gloo`` runs with
the CPU oracle as the per-shard compute.  Each rank owns half the KV heads
and their query heads, runs prefill + decode on its shard only, and the
layer output is reassembled by one all-gather; the result must equal the
single-process run over all heads bit-for-bit (KV heads are independent,
engine.py:126-132), and so must every index table and ledger
entry."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sparsekv_oracle as O
from paper_2502_14866_b200 import HeadProfile, classify_heads
from paper_2502_14866_b200.sharding import (HeadGather, shard_decode_inputs, shard_heads, shard_prefill_inputs,
                                            shard_profiles)

H, HKV, D, N = 8, 4, 32, 192
GATES = [0.9, 0.1, 0.8, 0.2, 0.05, 0.15, 0.12, 0.7]
CFG = dict(quant_bits=4, budget_tokens=128, reuse_interval=2, sink_blocks=1, local_blocks=1)
STEPS = 3


def _inputs():
    rng = np.random.default_rng(11)
    f = lambda *s: rng.standard_normal(s).astype(np.float16).astype(np.float32)  # noqa: E731
    q, k, v = f(N, H, D), f(N, HKV, D), f(N, HKV, D)
    dec = [(f(H, D), f(HKV, D), f(HKV, D)) for _ in range(STEPS)]
    return q, k, v, dec


def _roles(profiles):
    return [O.Role(p.head, p.gate, p.role, p.sink_blocks, p.local_blocks) for p in profiles]


def _full_run():
    q, k, v, dec = _inputs()
    eng = O.OracleEngine(O.Config(**CFG), O.assign_roles(GATES, 0.5, 1, 1))
    out = eng.prefill(q, k, v)
    steps = [eng.decode_step(*x) for x in dec]
    return out, steps


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q, k, v, dec = _inputs()
        shard = shard_heads(H, HKV, rank, world)
        prof = shard_profiles(classify_heads(GATES, 0.5, 1, 1), shard)
        eng = O.OracleEngine(O.Config(**CFG), _roles(prof))
        ql, kl, vl = shard_prefill_inputs(q, k, v, shard)
        local = torch.from_numpy(np.ascontiguousarray(eng.prefill(ql, kl, vl)))
        gather = HeadGather(world, N, shard.num_heads, D, torch.float32, "cpu")
        out = gather(local).numpy().copy()
        dgather = HeadGather(world, 1, shard.num_heads, D, torch.float32, "cpu")
        dec_out, tables = [], []
        for qn, kn, vn in dec:
            st = eng.decode_step(*shard_decode_inputs(qn, kn, vn, shard))
            dec_out.append(dgather(torch.from_numpy(st.output[None])).numpy()[0].copy())
            tbl = [None] * H
            dist.all_gather_object(tbl, st.tables)
            tables.append([t for part in tbl[:world] for t in part])
        if rank == 0:
            results.put((out, dec_out, tables))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_heads_partition():
    parts = [shard_heads(32, 8, r, 4) for r in range(4)]
    assert [(p.kv_begin, p.kv_end, p.q_begin, p.q_end) for p in parts] == [
        (0, 2, 0, 8), (2, 4, 8, 16), (4, 6, 16, 24), (6, 8, 24, 32)]
    assert sum(p.num_kv_heads for p in parts) == 8
    with pytest.raises(ValueError, match="multiple"):
        shard_heads(30, 8, 0, 2)
    with pytest.raises(ValueError, match="evenly"):
        shard_heads(32, 8, 0, 3)
    prof = shard_profiles(classify_heads([0.1 * i for i in range(8)], 0.5, 1, 2), shard_heads(8, 4, 1, 2))
    assert [p.head for p in prof] == [0, 1, 2, 3]
    assert all(isinstance(p, HeadProfile) for p in prof)


def test_gloo_world2_sharded_equals_unsharded():
    ctx = mp.get_context("spawn")
    results = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, results)) for r in range(2)]
    for p in procs:
        p.start()
    out, dec_out, tables = results.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref_out, ref_steps = _full_run()
    np.testing.assert_array_equal(out, ref_out)
    for i, st in enumerate(ref_steps):
        np.testing.assert_array_equal(dec_out[i], st.output)
        assert [tuple(t) for t in tables[i]] == [tuple(t) for t in st.tables]


def test_bench_gpus_2_launches_two_ranks():
    """`bench.py --gpus 2` without torchrun re-launches itself with 2 ranks
    (torch.distributed.run on 127.0.0.1); the ranks' KV-head shards, gathered
    over gloo, tile all 32 query / 8 KV heads."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    res = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--plan-only"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert res.returncode == 0, res.stderr[-3000:]
    line = [ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1]
    out = json.loads(line)
    assert out["world"] == 2 and out["covers_all_heads"]
    assert out["shards"] == [[0, 16, 0, 4], [16, 32, 4, 8]]
