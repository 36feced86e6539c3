"""K3 phase timeline from a -DSK_DEC_TIMING build (SK_LIB_PATH=tools/ab/lib_DT.so):
per-CTA globaltimer stamps of one decode_kernel launch at 128k (cfg2 layer),
warm and after an L2 flush.  Phases: 0 start, 1 header/selection/q loaded,
2 pages done, 3 CTA merge done, 4 cluster wait passed, 5 inbox complete, 6 end."""
import ctypes as C
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2502_14866_b200 as sk
from paper_2502_14866_b200 import _device, _lib
from paper_2502_14866_b200.selector import _Workspace

H, HKV, D, ctx = 32, 8, 128, 131072
lib = _lib.load()
GATES = [0.9 - 0.001 * h if h % 4 < 2 else 0.1 + 0.001 * h for h in range(H)]
e = sk.Engine(sk.EngineConfig(quant_bits=4, budget_tokens=4096, reuse_interval=4, local_blocks=4),
              sk.classify_heads(GATES, 0.5, 1, 4), device="cuda:0", capacity_tokens=ctx + 4096)
gen = torch.Generator(device="cuda").manual_seed(0)
k = torch.randn((ctx + 5, HKV, D), generator=gen, device="cuda", dtype=torch.float16)
e.load_context(k, k)
pool, g = e.cache.pool, e._group_size
q = torch.randn((H, D), device="cuda", dtype=torch.float16)
kn = torch.randn((HKV, D), device="cuda", dtype=torch.float16)
kp = int(os.environ.get('SK_KP', 64))
sel = torch.zeros((HKV, kp), dtype=torch.int32, device="cuda")
cnt = torch.zeros(HKV, dtype=torch.int32, device="cuda")
n_pages = -(-pool.tokens_host[0] // 64)
ws = _Workspace.get(pool.device, HKV, n_pages)
abi = pool.abi()
dws = pool.decode_workspace(g)
st = _device.stream_ptr(pool.device)
_lib.check(lib.sk_select_pages(C.byref(abi), HKV, g, q.data_ptr(), g * D, D, e._row_mask.data_ptr(),
                               pool.tokens.data_ptr(), None, kp, n_pages, sel.data_ptr(), cnt.data_ptr(), kp,
                               ws.data_ptr(), ws.numel(), 0, st))
out = torch.empty((H, D), dtype=torch.float16, device="cuda")


def dec():
    _lib.check(lib.sk_decode_attn(C.byref(abi), HKV, g, q.data_ptr(), g * D, D, kn.data_ptr(), kn.data_ptr(), D,
                                  e._row_mask.data_ptr(), None, sel.data_ptr(), cnt.data_ptr(), kp,
                                  pool.tokens.data_ptr(), C.c_float(1 / math.sqrt(D)), out.data_ptr(), g * D, D,
                                  _lib.SK_F16, 0, dws.data_ptr(), dws.numel(), st))


flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
buf = np.zeros((4096, 8), np.uint64)
for label in ("warm", "cold", "warm", "cold"):
    for _ in range(300):
        dec()
    buf[:] = 0
    lib.sk_debug_decode_stamps_clear()
    if label == "cold":
        flush.zero_()
    dec()
    torch.cuda.synchronize()
    assert lib.sk_debug_decode_stamps(buf.ctypes.data_as(C.c_void_p)) == 0
    t = buf[:4000].astype(np.int64)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    rel = np.where(t > 0, (t - t0) / 1000.0, np.nan)
    last = ~np.isnan(rel[:, 6])
    print(label, "ctas", len(t), "start spread %.2f us" % np.nanmax(rel[:, 0]),
          "| header %.2f units %.2f cta-merge %.2f ticket %.2f" % tuple(np.nanmean(np.diff(rel[:, :5], axis=1), 0)),
          "| last CTA: partials %.2f finish %.2f end %.2f" % (np.nanmean(rel[last, 5] - rel[last, 4]),
                                                            np.nanmean(rel[last, 6] - rel[last, 5]),
                                                            np.nanmax(rel[last, 6])))
    w = buf[4000:4008, :4].astype(np.int64)
    w = w[w[:, 0] > 0]
    if len(w):
        print("   unit compute: %.2f us, %d cycles (%.2f GHz); compute starts %.2f us after CTA start" % (
            np.mean(w[:, 2] - w[:, 0]) / 1000.0, np.mean(w[:, 3] - w[:, 1]),
            np.mean(w[:, 3] - w[:, 1]) / np.mean(w[:, 2] - w[:, 0]), (w[:, 0].min() - t0) / 1000.0))
