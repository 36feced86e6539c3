"""Multi-layer prefill from host buffers with the PCIe copies overlapped (an
extension: the reference API is one synchronous ``Engine.prefill`` per
layer, engine.py:136-173).

A host caller that keeps q/k/v in (pinned) host memory pays, per layer, an
upload of q/k/v and a download of the output.  Calling ``Engine.prefill``
layer by layer serialises those copies with the attention kernels.
``prefill_layers`` runs the same per-layer work -- ``Engine.prefill_device``
(K4 + K1) on each layer's engine -- but uploads layer l+1 on one copy stream
and downloads layer l-1 on another while layer l computes, with two device
input buffers in flight.  Outputs and caches are bit-identical to the
sequential calls (tests/test_gpu_pipeline.py).  Inputs are checked for
non-finite values on the device; the check is read once at the end, so a
bad layer raises after the pipeline drains rather than before it runs.
"""

from __future__ import annotations

from typing import Sequence

import torch

from . import _device


def prefill_layers(engines: Sequence, inputs: Sequence, outputs: Sequence) -> None:
    """engines[l].prefill on host tensors: inputs[l] = (q [N,H,D], k [S,Hkv,D],
    v [S,Hkv,D]) and outputs[l] [N,H,D], all CPU torch tensors (pinned for
    asynchronous copies) in the engines' dtype.  Returns when every output
    has landed in host memory."""
    n_layers = len(engines)
    if not (len(inputs) == len(outputs) == n_layers) or n_layers == 0:
        raise ValueError("need one (q, k, v) input and one output per engine")
    dev = engines[0].device
    dt = engines[0]._dtype
    q0, k0, _ = inputs[0]
    n, h, d = q0.shape
    s, hkv, _ = k0.shape
    dp = _device.padded_dim(d)
    for q, k, v in inputs:
        if tuple(q.shape) != (n, h, d) or tuple(k.shape) != (s, hkv, d) or tuple(v.shape) != (s, hkv, d):
            raise ValueError("every layer must have the same q/k/v shapes")
        if q.is_cuda or k.is_cuda or v.is_cuda or q.dtype != dt or k.dtype != dt or v.dtype != dt:
            raise ValueError(f"inputs must be host tensors of the engines' dtype {dt}")
    for o in outputs:
        if o.is_cuda or tuple(o.shape) != (n, h, d) or o.dtype != dt:
            raise ValueError("outputs must be host tensors [N, H, D] of the engines' dtype")
    comp = torch.cuda.current_stream(dev)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    bufs = [(torch.zeros((n, h, dp), dtype=dt, device=dev), torch.zeros((s, hkv, dp), dtype=dt, device=dev),
             torch.zeros((s, hkv, dp), dtype=dt, device=dev)) for _ in range(2)]
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_used = [torch.cuda.Event() for _ in range(2)]
    bad = torch.zeros(n_layers, dtype=torch.bool, device=dev)
    s_in.wait_stream(comp)  # the zero-filled buffers are ready

    def upload(layer: int) -> None:
        b = layer % 2
        with torch.cuda.stream(s_in):
            if layer >= 2:
                s_in.wait_event(ev_used[b])  # layer-2 has consumed this buffer
            for dst, src in zip(bufs[b], inputs[layer]):
                dst[..., :d].copy_(src, non_blocking=True)
            ev_in[b].record(s_in)

    upload(0)
    for layer in range(n_layers):
        if layer + 1 < n_layers:
            upload(layer + 1)
        b = layer % 2
        comp.wait_event(ev_in[b])
        q, k, v = bufs[b]
        bad[layer] = ~(_device.all_finite(q) & _device.all_finite(k) & _device.all_finite(v))
        out = engines[layer].prefill_device(q, k, v, d)
        ev_used[b].record(comp)
        with torch.cuda.stream(s_out):
            s_out.wait_stream(comp)
            outputs[layer].copy_(out[..., :d], non_blocking=True)
            out.record_stream(s_out)
    comp.wait_stream(s_out)
    comp.wait_stream(s_in)
    flags = bad.cpu()  # waits for everything queued above
    if bool(flags.any()):
        raise ValueError(f"non-finite values in the inputs of layer(s) {flags.nonzero().flatten().tolist()}")
