"""Phase-B stamps of a -DSK_SEL_TIMING K2 build (SK_LIB_PATH=tools/ab/lib_T.so):
globaltimer deltas (ns) between the checkpoints of topk_filtered."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
def launch():
    _lib.check(lib.sk_select_pages(C.byref(abi), HKV, g, q.data_ptr(), g * D, D, e._row_mask.data_ptr(),
                                   pool.tokens.data_ptr(), None, kp, n_pages, sel.data_ptr(), cnt.data_ptr(), kp,
                                   ws.data_ptr(), ws.numel(), 0, _device.stream_ptr(pool.device)))


for it in range(3):
    for _ in range(300):  # back-to-back launches: clocks ramped up as in the graph probes
        launch()
    torch.cuda.synchronize()
    off = lib.sk_select_scores_offset(HKV) + 8 * HKV * n_pages
    st = ws[off:off + 8 * HKV * n_pages].view(torch.int64).view(HKV, n_pages)[:, :6].cpu()
    for s in range(HKV):
        t = st[s].tolist()
        print(it, s, [t[i + 1] - t[i] for i in range(5)], "total", t[5] - t[0])
    import numpy as np
    ph = ws[off:off + 8 * HKV * n_pages].view(torch.int64).view(HKV, n_pages)[:, 8:8 + 3 * 64].cpu().numpy()
    ph = ph.reshape(HKV, -1, 3)
    ph = ph[ph[:, :, 0] > 0]
    t0 = ph[:, 0].min()
    print(it, "phase A over %d CTAs: start spread %.2f us, prologue %.2f us, tiles %.2f us (max end %.2f us)" % (
        len(ph), (ph[:, 0].max() - t0) / 1e3, np.mean(ph[:, 1] - ph[:, 0]) / 1e3, np.mean(ph[:, 2] - ph[:, 1]) / 1e3,
        (ph[:, 2].max() - t0) / 1e3))
    b0 = st[:, 0].numpy()
    b5 = st[:, 5].numpy()
    print(it, "phase B (last CTAs): start %.2f..%.2f us, end %.2f us after the first CTA's start" % (
        (b0.min() - t0) / 1e3, (b0.max() - t0) / 1e3, (b5.max() - t0) / 1e3))
