"""Where the host-buffer prefill time goes: 8 layers at 128k (cfg2 heads),
ms per layer for the device-only loop, prefill_layers (overlapped copies)
and the sequential public API; then one prefill_layers pass under
torch.cuda.set_sync_debug_mode('warn') to list implicit host syncs."""
import os
import sys
import time
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2502_14866_b200 as sk

L, N, H, HKV, D = 8, 131072, 32, 8, 128
gates = [0.9 - 0.001 * i if i % 4 < 2 else 0.1 + 0.001 * i for i in range(H)]
prof = sk.classify_heads(gates, 0.5, 1, 4)
cfg = sk.EngineConfig(local_blocks=4)
engines = [sk.Engine(cfg, prof, device="cuda:0", capacity_tokens=N + 8) for _ in range(L)]
qh = torch.randn((N, H, D), dtype=torch.float16).pin_memory()
kh = torch.randn((N, HKV, D), dtype=torch.float16).pin_memory()
vh = torch.randn((N, HKV, D), dtype=torch.float16).pin_memory()
oh = torch.empty((N, H, D), dtype=torch.float16).pin_memory()
qd, kd, vd = qh.cuda(), kh.cuda(), vh.cuda()


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / L


dev_only = lambda: [e.prefill_device(qd, kd, vd, D) for e in engines]  # noqa: E731
pipe = lambda: sk.prefill_layers(engines, [(qh, kh, vh)] * L, [oh] * L)  # noqa: E731


def seq():
    for e in engines:
        oh.copy_(e.prefill(sk.Workload(qh, kh, vh)), non_blocking=True)


for name, fn in (("device-only", dev_only), ("prefill_layers", pipe), ("sequential", seq)):
    fn()
    print(f"{name}: {min(timed(fn) for _ in range(2)):.1f} ms/layer", flush=True)
torch.cuda.set_sync_debug_mode("warn")
with warnings.catch_warnings(record=True) as w:
    warnings.simplefilter("always")
    pipe()
    torch.cuda.set_sync_debug_mode(0)
for x in w[:20]:
    print("SYNC:", str(x.message)[:200], x.filename.split("/")[-1], x.lineno)


# ---- timeline: the prefill_layers schedule with events on every stream ----
def traced():
    dev = torch.device("cuda:0")
    comp = torch.cuda.current_stream(dev)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    bufs = [(torch.zeros((N, H, D), dtype=torch.float16, device=dev), torch.zeros((N, HKV, D), dtype=torch.float16,
             device=dev), torch.zeros((N, HKV, D), dtype=torch.float16, device=dev)) for _ in range(2)]
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_used = [torch.cuda.Event() for _ in range(2)]
    T = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    marks = []
    t0 = T()
    t0.record(comp)
    s_in.wait_stream(comp)

    def upload(layer):
        b = layer % 2
        with torch.cuda.stream(s_in):
            if layer >= 2:
                s_in.wait_event(ev_used[b])
            a = T(); a.record(s_in)
            for dst, src in zip(bufs[b], (qh, kh, vh)):
                dst.copy_(src, non_blocking=True)
            z = T(); z.record(s_in)
            marks.append(("up", layer, a, z))
            ev_in[b].record(s_in)

    upload(0)
    for layer in range(L):
        if layer + 1 < L:
            upload(layer + 1)
        b = layer % 2
        comp.wait_event(ev_in[b])
        a = T(); a.record(comp)
        out = engines[layer].prefill_device(*bufs[b], D)
        z = T(); z.record(comp)
        marks.append(("comp", layer, a, z))
        ev_used[b].record(comp)
        with torch.cuda.stream(s_out):
            s_out.wait_stream(comp)
            a2 = T(); a2.record(s_out)
            oh.copy_(out, non_blocking=True)
            z2 = T(); z2.record(s_out)
            marks.append(("down", layer, a2, z2))
            out.record_stream(s_out)
    comp.wait_stream(s_out)
    torch.cuda.synchronize()
    for kind, layer, a, z in marks:
        print(f"{kind:5s} L{layer}: {t0.elapsed_time(a):8.1f} -> {t0.elapsed_time(z):8.1f} ms")


traced()
traced()
