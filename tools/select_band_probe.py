"""K2 phase-A diagnostics on the cfg2 layer (128k, 8 KV heads, balanced
gates): per stream the fp32 scores / bounds the kernel stored, the exact
fp64 scores (sk_score_pages), the largest |approx - exact| / bound, and the
band size around the K-th score that phase B has to rescore."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2502_14866_b200 as sk
from paper_2502_14866_b200 import _device, _lib
from paper_2502_14866_b200.selector import _Workspace

H, HKV, D, ctx = 32, 8, 128, 131072
GATES = [0.9 - 0.001 * h if h % 4 < 2 else 0.1 + 0.001 * h for h in range(H)]
e = sk.Engine(sk.EngineConfig(quant_bits=4, budget_tokens=4096, reuse_interval=4, local_blocks=4),
              sk.classify_heads(GATES, 0.5, 1, 4), device="cuda:0", capacity_tokens=ctx + 64)
gen = torch.Generator(device="cuda").manual_seed(0)
k = torch.randn((ctx, HKV, D), generator=gen, device="cuda", dtype=torch.float16)
e.load_context(k, k)
pool, g = e.cache.pool, e._group_size
q = torch.randn((HKV * g, D), device="cuda", dtype=torch.float16)
n_pages, kp = 2048, 64
sel = torch.zeros((HKV, kp), dtype=torch.int32, device="cuda")
cnt = torch.zeros(HKV, dtype=torch.int32, device="cuda")
ws = _Workspace.get(pool.device, HKV, n_pages)
lib = _lib.load()
abi = pool.abi()
st = _device.stream_ptr(pool.device)
_lib.check(lib.sk_select_pages(C.byref(abi), HKV, g, q.data_ptr(), g * D, D, e._row_mask.data_ptr(),
                               pool.tokens.data_ptr(), None, kp, n_pages, sel.data_ptr(), cnt.data_ptr(), kp,
                               ws.data_ptr(), ws.numel(), 0, st))
exact = torch.empty((HKV, n_pages), dtype=torch.float64, device="cuda")
_lib.check(lib.sk_score_pages(C.byref(abi), HKV, g, q.data_ptr(), g * D, D, e._row_mask.data_ptr(),
                              pool.tokens.data_ptr(), exact.data_ptr(), n_pages, st))
torch.cuda.synchronize()
off = lib.sk_select_scores_offset(HKV)
pairs = ws[off:off + 8 * HKV * n_pages].view(torch.float32).view(HKV, n_pages, 2).double().cpu().numpy()
ex = exact.cpu().numpy()
for s in range(HKV):
    a, err, x = pairs[s, :, 0], pairs[s, :, 1], ex[s]
    pins = {0, n_pages - 2, n_pages - 1}
    cand = np.array([i for i in range(n_pages) if i not in pins])
    if not np.isfinite(x[cand]).all():
        continue
    E = err[cand].max()
    T = np.sort(a[cand])[::-1][kp - 3 - 1]
    band = int((np.abs(a[cand] - T) <= 2 * E).sum())
    print(json.dumps({"stream": s, "E": float(E), "max_abs_err": float(np.abs(a - x)[cand].max()),
                      "max_err_over_bound": float((np.abs(a - x) / err)[cand].max()), "T": float(T),
                      "band": band, "score_std": float(a[cand].std())}))
