"""Chains of decode-step kernels over SK_LAYERS layers (cfg2 heads, 128k),
captured in one CUDA graph, with and without programmatic dependent launch:
  reuse step     = K3(0) K3(1) ...                 (selection ready)
  selection step = K2(0) K3(0) K2(1) K3(1) ...
L2 flushed before each replay; prints us per layer."""
import ctypes as C
import math
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2502_14866_b200 as sk
from paper_2502_14866_b200 import _lib
from paper_2502_14866_b200.selector import _Workspace

L, N, H, HKV, D = int(os.environ.get("SK_LAYERS", 8)), 131072, 32, 8, 128
lib = _lib.load()
gates = [0.9 - 0.001 * i if i % 4 < 2 else 0.1 + 0.001 * i for i in range(H)]
prof = sk.classify_heads(gates, 0.5, 1, 4)
cfg = sk.EngineConfig(local_blocks=4)
g = torch.Generator(device="cuda").manual_seed(0)
engines = []
for _ in range(L):
    e = sk.Engine(cfg, prof, device="cuda:0", capacity_tokens=N + 64)
    k = torch.randn((N, HKV, D), generator=g, device="cuda", dtype=torch.float16)
    e.load_context(k, k)
    engines.append(e)
grp = H // HKV
q = torch.randn((L, H, D), generator=g, device="cuda", dtype=torch.float16)
kn = torch.randn((L, HKV, D), generator=g, device="cuda", dtype=torch.float16)
out = torch.empty((L, H, D), device="cuda", dtype=torch.float16)
kp = 64
sel = [torch.zeros((HKV, kp), dtype=torch.int32, device="cuda") for _ in range(L)]
cnt = [torch.zeros(HKV, dtype=torch.int32, device="cuda") for _ in range(L)]
n_pages = -(-N // 64)
ws = [torch.zeros(lib.sk_select_workspace(HKV, n_pages), dtype=torch.uint8, device="cuda") for _ in range(L)]


def launch(li, select, pdl):
    e = engines[li]
    pool = e.cache.pool
    abi = pool.abi()
    st = torch.cuda.current_stream().cuda_stream
    if select:
        _lib.check(lib.sk_select_pages(C.byref(abi), HKV, grp, q[li].data_ptr(), grp * D, D, e._row_mask.data_ptr(),
                                       pool.tokens.data_ptr(), None, kp, n_pages, sel[li].data_ptr(),
                                       cnt[li].data_ptr(), kp, ws[li].data_ptr(), ws[li].numel(),
                                       _lib.SK_LAUNCH_PDL if pdl else 0, st))
    flags = (_lib.SK_LAUNCH_PDL | (0 if select else _lib.SK_DECODE_SEL_READY)) if pdl else 0
    dws = pool.decode_workspace(grp)
    _lib.check(lib.sk_decode_attn(C.byref(abi), HKV, grp, q[li].data_ptr(), grp * D, D, kn[li].data_ptr(),
                                  kn[li].data_ptr(), D, e._row_mask.data_ptr(), None, sel[li].data_ptr(),
                                  cnt[li].data_ptr(), kp, pool.tokens.data_ptr(), C.c_float(1 / math.sqrt(D)),
                                  out[li].data_ptr(), grp * D, D, _lib.SK_F16, flags, dws.data_ptr(), dws.numel(),
                                  st))


for li in range(L):
    launch(li, True, False)
torch.cuda.synchronize()
ref = out.clone()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for select in (False, True):
    for pdl in (False, True):
        gr = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(gr, stream=s):
                for li in range(L):
                    launch(li, select, pdl)
        torch.cuda.current_stream().wait_stream(s)
        ts = []
        for _ in range(20):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            gr.replay()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        same = bool(torch.equal(out, ref))
        print(f"{'selection' if select else 'reuse':9s} step pdl={int(pdl)}: {statistics.median(ts) / L:6.2f} us/layer"
              f" (same output as eager: {same})", flush=True)
