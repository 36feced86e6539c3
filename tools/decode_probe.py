"""Isolate decode/select kernel costs at 128k: CUDA-event timing of the raw
ABI calls with features toggled (fused append on/off, streaming rows on/off,
pages per split)."""
import ctypes as C
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2502_14866_b200 as sk
from paper_2502_14866_b200 import _device, _lib
from paper_2502_14866_b200.selector import _Workspace

ctx = int(os.environ.get("SK_CTX", 131072))
H, HKV, D = 32, 8, 128
lib = _lib.load()


def make(gates):
    cfg = sk.EngineConfig(quant_bits=4, budget_tokens=int(os.environ.get("SK_BUDGET", 4096)), reuse_interval=4,
                          local_blocks=4)
    prof = sk.classify_heads(gates, 0.5 if len(set(gates)) > 1 else 0.0, 1, 4)
    e = sk.Engine(cfg, prof, device="cuda:0", capacity_tokens=ctx + 4096)
    g = torch.Generator(device="cuda").manual_seed(0)
    k = torch.randn((ctx + 5, HKV, D), generator=g, device="cuda", dtype=torch.float16)
    e.load_context(k, k)
    return e


def time_it(fn, n=32):
    """Per-call device time of n calls captured in one CUDA graph (no host
    launch overhead in the measurement; L2 warm after the first call)."""
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
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (5 * n) * 1e3


tiny = torch.zeros(1, device="cuda")
print("graph node floor (1-element torch add) us", round(time_it(lambda: tiny.add_(1)), 2), flush=True)

for name, gates in [("balanced", [0.9 - 0.001 * h if h % 4 < 2 else 0.1 + 0.001 * h for h in range(H)]),
                    ("all-retrieval", [0.9] * H)]:
    e = make(gates)
    pool = e.cache.pool
    g = e._group_size
    q = torch.randn((H, D), device="cuda", dtype=torch.float16)
    kn = torch.randn((HKV, D), device="cuda", dtype=torch.float16)
    kp = 64
    sel = torch.zeros((HKV, kp), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(HKV, dtype=torch.int32, device="cuda")
    n_pages = -(-pool.tokens_host[0] // 64)
    ws = _Workspace.get(pool.device, HKV, n_pages)
    abi = pool.abi()
    dws = pool.decode_workspace(g)

    def sel_call():
        rc = lib.sk_select_pages(C.byref(abi), HKV, g, q.data_ptr(), g * D, D, e._row_mask.data_ptr(),
                                 pool.tokens.data_ptr(), None, kp, n_pages, sel.data_ptr(), cnt.data_ptr(), kp,
                                 ws.data_ptr(), ws.numel(), 0, torch.cuda.current_stream().cuda_stream)
        _lib.check(rc)

    print(name, "select us", round(time_it(sel_call), 2))
    for fuse in (0, 1):
        out = torch.empty((H, D), dtype=torch.float16, device="cuda")

        def dec_call():
            rc = lib.sk_decode_attn(C.byref(abi), HKV, g, q.data_ptr(), g * D, D, kn.data_ptr(), kn.data_ptr(), D,
                                    e._row_mask.data_ptr(), None, sel.data_ptr(), cnt.data_ptr(), kp,
                                    pool.tokens.data_ptr(), C.c_float(1 / math.sqrt(D)), out.data_ptr(), g * D, D,
                                    _lib.SK_F16, fuse, dws.data_ptr(), dws.numel(), torch.cuda.current_stream().cuda_stream)
            _lib.check(rc)

        print(name, f"decode append={fuse} us", round(time_it(dec_call), 2))
