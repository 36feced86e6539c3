"""K2 (sk_select_pages) timing probe: warm (32 back-to-back calls in one CUDA
graph) and cold (each call behind a 256 MB L2 flush; a graph of N x (flush +
select) minus a graph of N x flush) for the cfg2 layer (128k, 8 KV heads,
balanced gates) and the cfg4 batched layer (16 x 64k).  Prints JSON lines."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2502_14866_b200 as sk
from paper_2502_14866_b200 import _lib
from paper_2502_14866_b200.batch import BatchedLayer
from paper_2502_14866_b200.selector import _Workspace

H, HKV, D = 32, 8, 128
lib = _lib.load()
GATES = [0.9 - 0.001 * h if h % 4 < 2 else 0.1 + 0.001 * h for h in range(H)]
CFG = sk.EngineConfig(quant_bits=4, budget_tokens=4096, reuse_interval=4, local_blocks=4)
PROF = sk.classify_heads(GATES, 0.5, 1, 4)


def graph_of(fn, n):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    return g


def replay_us(g, n, reps=5):
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (reps * n) * 1e3


def probe(name, pool, row_mask, n_streams, g):
    q = torch.randn((n_streams * g, D), device="cuda", dtype=torch.float16)
    kp = 64
    sel = torch.zeros((n_streams, kp), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(n_streams, dtype=torch.int32, device="cuda")
    n_pages = -(-max(pool.tokens_host) // 64)
    ws = _Workspace.get(pool.device, n_streams, n_pages)
    abi = pool.abi()

    def sel_call():
        rc = lib.sk_select_pages(C.byref(abi), n_streams, g, q.data_ptr(), g * D, D, row_mask.data_ptr(),
                                 pool.tokens.data_ptr(), None, kp, n_pages, sel.data_ptr(), cnt.data_ptr(), kp,
                                 ws.data_ptr(), ws.numel(), 0, torch.cuda.current_stream().cuda_stream)
        _lib.check(rc)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    n = 16
    warm = replay_us(graph_of(sel_call, 32), 32)
    g_fs = graph_of(lambda: (flush.zero_(), sel_call()), n)
    g_f = graph_of(lambda: flush.zero_(), n)
    cold = replay_us(g_fs, n) - replay_us(g_f, n)
    stats_bytes = n_streams * n_pages * 4 * 2 * D * 2
    print(json.dumps({"case": name, "streams": n_streams, "pages": n_pages, "warm_us": round(warm, 2),
                      "cold_us": round(cold, 2), "stats_MB": round(stats_bytes / 1e6, 2),
                      "cold_GBps": round(stats_bytes / cold / 1e3, 1)}), flush=True)


def main():
    which = sys.argv[1:] or ["cfg2", "cfg4"]
    if "cfg2" in which:
        ctx = 131072
        e = sk.Engine(CFG, PROF, device="cuda:0", capacity_tokens=ctx + 64)
        gen = torch.Generator(device="cuda").manual_seed(0)
        k = torch.randn((ctx, HKV, D), generator=gen, device="cuda", dtype=torch.float16)
        e.load_context(k, k)
        del k
        probe("cfg2 128k x 8 streams", e.cache.pool, e._row_mask, HKV, e._group_size)
    if "cfg4" in which:
        B, ctx = 16, 65536
        ly = BatchedLayer(CFG, PROF, B, HKV, D, device="cuda:0", capacity_tokens=ctx + 64)
        gen = torch.Generator(device="cuda").manual_seed(1)
        for b in range(B):
            k = torch.randn((ctx, HKV, D), generator=gen, device="cuda", dtype=torch.float16)
            ly.load_context(b, k, k)
        probe("cfg4 16 x 64k (128 streams)", ly.pool, ly._row_mask, B * HKV, HKV and H // HKV)


if __name__ == "__main__":
    main()
