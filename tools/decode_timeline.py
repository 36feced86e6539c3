"""Phase timeline of the decode kernel (library built with -DSK_DECODE_TIMING):
%globaltimer stamps per CTA of stream 0, relative to the first CTA start."""
import ctypes as C
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
np.set_printoptions(linewidth=220, suppress=True)
import torch

import paper_2502_14866_b200 as sk
from paper_2502_14866_b200 import _lib
from paper_2502_14866_b200.selector import _Workspace

ctx = 131072
H, HKV, D = 32, 8, 128
gates = [0.9 - 0.001 * h if h % 4 < 2 else 0.1 + 0.001 * h for h in range(H)]
cfg = sk.EngineConfig(quant_bits=4, budget_tokens=4096, reuse_interval=4, local_blocks=4)
e = sk.Engine(cfg, sk.classify_heads(gates, 0.5, 1, 4), device="cuda:0", capacity_tokens=ctx + 4096)
g = torch.Generator(device="cuda").manual_seed(0)
k = torch.randn((ctx + 5, HKV, D), generator=g, device="cuda", dtype=torch.float16)
e.load_context(k, k)
lib = _lib.load()
lib.sk_debug_decode_times.argtypes = [C.c_void_p]
pool = e.cache.pool
st = torch.cuda.current_stream().cuda_stream
q = torch.randn((H, D), device="cuda", dtype=torch.float16)
sel = torch.zeros((HKV, 64), dtype=torch.int32, device="cuda")
cnt = torch.zeros(HKV, dtype=torch.int32, device="cuda")
n_pages = -(-pool.tokens_host[0] // 64)
ws = _Workspace.get(pool.device, HKV, n_pages)
abi = pool.abi()
_lib.check(lib.sk_select_pages(C.byref(abi), HKV, 4, q.data_ptr(), 4 * D, D, e._row_mask.data_ptr(),
                               pool.tokens.data_ptr(), None, 64, n_pages, sel.data_ptr(), cnt.data_ptr(), 64,
                               ws.data_ptr(), ws.numel(), st))
names = ["start", "prologue", "staged", "items", "merged", "preticket", "ticket", "hdr", "selstg", "sync1", "tables"] + [f"w{i}" for i in range(8)]
for pps in (2, 4):
    ms = -(-69 // pps)
    wsd = torch.zeros(lib.sk_decode_workspace(HKV, 4, D, ms), dtype=torch.uint8, device="cuda")
    out = torch.empty((H, D), dtype=torch.float16, device="cuda")
    for rep in range(3):
        _lib.check(lib.sk_decode_attn(C.byref(abi), HKV, 4, q.data_ptr(), 4 * D, D, k[0].data_ptr(), k[1].data_ptr(),
                                      D, e._row_mask.data_ptr(), sel.data_ptr(), cnt.data_ptr(), 64,
                                      pool.tokens.data_ptr(), C.c_float(1 / math.sqrt(D)), out.data_ptr(), 4 * D, D,
                                      _lib.SK_F16, pps, ms, 0, wsd.data_ptr(), wsd.numel(), st))
        torch.cuda.synchronize()
    buf = np.zeros((64, 32), np.uint64)
    assert lib.sk_debug_decode_times(buf.ctypes.data) == 0
    n = int((buf[:, 0] > 0).sum())
    t0 = int(buf[:n, 0].min())
    rel = (buf[:n].astype(np.int64) - t0) / 1000.0
    rel[buf[:n] == 0] = np.nan
    print(f"pps={pps} CTAs(stream0)={n}  columns: {names}")
    for i in range(0, n, max(1, n // 5)):
        print("  cta", i, np.round(rel[i, :19], 2))
    print("  median", np.round(np.nanmedian(rel[:, :19], axis=0), 2))
    print("  max   ", np.round(np.nanmax(rel[:, :19], axis=0), 2))
