"""CUDA-graph decode over many layers (extension outside the reference API).

A decode step of a model runs every layer's attention: K2 selection (only
on reuse-window starts) and K3 split-KV decode with the fused append.  At
128k context one layer's kernels take a few microseconds, so Python launch
overhead would dominate; this runner captures the whole multi-layer step
into two CUDA graphs (selection step / reuse step) over static buffers and
replays them.  Inside a graph the kernels chain by programmatic dependent
launch, and the one-token appends of every `append_group` layers run as one
launch on a side stream, overlapping the following layers' attention.
Token counters, page tables and workspaces are device
resident, so replays need no host->device traffic besides the new q/k/v
rows.  Per-engine host bookkeeping (token mirrors, step counters, ledger)
is advanced exactly like Engine.decode_step would.

Multi-GPU (KV-head sharding): with `group`, each layer's head
outputs are all-gathered over NCCL right behind that layer's K3, inside the
captured graph (one collective per layer, at the layer boundary), into
`gathered[layer]` = [world, H/world, Dp] head-major.
"""

from __future__ import annotations

import ctypes as C
import math

import torch

from . import _device, _lib
from .engine import DECODE, Engine
from .heads import RETRIEVAL, lambda_segments
from .selector import _Workspace, selection_size


class DecodeGraph:
    def __init__(self, engines: list, max_steps: int, head_dim: int, record_ledger: bool = True, group=None,
                 append_group: int = 8):
        if not engines:
            raise ValueError("need at least one engine")
        if record_ledger and any(not hasattr(e, "_plans") for e in engines):
            raise ValueError("per-head ledgers are recorded for single-sequence Engines only")
        e0 = engines[0]
        self.engines = engines
        self.cfg = e0.config
        self.dev = e0.device
        self.head_dim = head_dim
        self.record_ledger = record_ledger
        self.append_group = max(1, int(append_group))  # layers per K1 append launch
        pools = [e.cache.pool for e in engines]
        # streams may hold different token counts (a ragged batch: per-sequence
        # page tables); every layer must hold the same counts stream by stream
        start = list(pools[0].tokens_host)
        for p in pools:
            if list(p.tokens_host) != start:
                raise ValueError("all layers must hold the same token counts, stream by stream")
        tok = max(start)
        for p in pools:
            p.reserve(tok + max_steps + 1)
        self.pools = pools
        for e in engines:  # a streaming pool never holds more than its own window
            if getattr(e, "_row_window", None) is not None and hasattr(e, "_check_windows"):
                e._check_windows(-(-(tok + max_steps) // e.config.physical_page))
        self.g = e0._group_size
        self.h_kv = pools[0].n_streams
        self.h = self.h_kv * self.g
        self.dp = pools[0].Dp
        self.dtype = pools[0].dtype
        self.start_tokens = tok
        self.start_per_stream = start
        self.steps_done = 0
        self._valid = None  # cached [lo, hi) of steps the current selections cover
        self._next_step = -1
        self.max_steps = max_steps
        cfg = self.cfg
        self.k_pages = -(-cfg.budget_tokens // cfg.physical_page)
        self.max_pages_hint = -(-(tok + max_steps) // cfg.physical_page)
        L = len(engines)
        z = lambda *s, dt=self.dtype: torch.zeros(*s, dtype=dt, device=self.dev)  # noqa: E731
        self.q = z(L, self.h, self.dp)
        self.k = z(L, self.h_kv, self.dp)
        self.v = z(L, self.h_kv, self.dp)
        self.out = z(L, self.h, self.dp)
        width = max(4, self.k_pages)
        self.sel = [torch.zeros((self.h_kv, width), dtype=torch.int32, device=self.dev) for _ in engines]
        self.cnt = [torch.zeros(self.h_kv, dtype=torch.int32, device=self.dev) for _ in engines]
        self.sel_ws = [torch.zeros(_lib.load().sk_select_workspace(self.h_kv, self.max_pages_hint),
                                   dtype=torch.uint8, device=self.dev) for _ in engines]
        self.graphs = {}
        self.group = group
        self.gathered = None
        if group is not None:
            import torch.distributed as dist
            world = dist.get_world_size(group)
            self.gathered = torch.zeros((L, world) + tuple(self.out.shape[1:]), dtype=self.dtype, device=self.dev)
            dist.all_gather_into_tensor(self.gathered[0], self.out[0], group=group)  # communicator up before capture
            torch.cuda.synchronize(self.dev)
        self._side = torch.cuda.Stream(device=self.dev)
        # prime selections (first step must select anyway) then capture
        self._capture()

    # -- launches ---------------------------------------------------------------
    def _launch_layer(self, li: int, select: bool, side) -> None:
        e, pool = self.engines[li], self.pools[li]
        lib = _lib.load()
        main = torch.cuda.current_stream(self.dev)
        stream = main.cuda_stream
        abi = pool.abi()
        if select:
            ws = self.sel_ws[li]
            rc = lib.sk_select_pages(C.byref(abi), self.h_kv, self.g, self.q[li].data_ptr(), self.g * self.dp,
                                     self.dp, e._row_mask.data_ptr(), pool.tokens.data_ptr(), None, self.k_pages,
                                     self.max_pages_hint, self.sel[li].data_ptr(), self.cnt[li].data_ptr(),
                                     self.sel[li].shape[1], ws.data_ptr(), ws.numel(), _lib.SK_LAUNCH_PDL, stream)
            _lib.check(rc)
        dws = pool.decode_workspace(self.g)
        # programmatic dependent launches: each kernel's prologue (page table, the
        # pages themselves, and on reuse steps the selection) overlaps the previous
        # kernel's tail; q / the new token are read after the dependency wait
        flags = _lib.SK_LAUNCH_PDL | (0 if select else _lib.SK_DECODE_SEL_READY)
        rc = lib.sk_decode_attn(C.byref(abi), self.h_kv, self.g, self.q[li].data_ptr(), self.g * self.dp, self.dp,
                                self.k[li].data_ptr(), self.v[li].data_ptr(), self.dp, e._row_mask.data_ptr(),
                                e.row_window_ptr(), self.sel[li].data_ptr(), self.cnt[li].data_ptr(),
                                self.sel[li].shape[1], pool.tokens.data_ptr(),
                                C.c_float(1.0 / math.sqrt(self.head_dim)), self.out[li].data_ptr(),
                                self.g * self.dp, self.dp, _device.sk_dtype(self.dtype), flags, dws.data_ptr(),
                                dws.numel(), stream)
        _lib.check(rc)
        if self.group is not None:  # layer boundary: head outputs of every rank
            import torch.distributed as dist
            dist.all_gather_into_tensor(self.gathered[li], self.out[li], group=self.group)

    def _launch_appends(self, l0: int, l1: int, side) -> None:
        """K1 one-token appends of layers [l0, l1) in one launch on the side
        stream, behind those layers' attention: it overlaps the next layers'."""
        n = l1 - l0
        pools = (_lib.SkPool * n)(*[self.pools[li].abi() for li in range(l0, l1)])
        toks = (C.c_void_p * n)(*[self.pools[li].tokens.data_ptr() for li in range(l0, l1)])
        side.wait_stream(torch.cuda.current_stream(self.dev))
        rc = _lib.load().sk_append_token_layers(pools, n, self.h_kv, self.k[l0].data_ptr(), self.v[l0].data_ptr(),
                                                self.h_kv * self.dp, self.dp, toks, side.cuda_stream)
        _lib.check(rc)

    def _launch_step(self, select: bool) -> None:
        main = torch.cuda.current_stream(self.dev)
        side = self._side
        L, l0 = len(self.engines), 0
        for li in range(L):
            self._launch_layer(li, select, side)
            if li + 1 - l0 == self.append_group or li == L - 1:
                self._launch_appends(l0, li + 1, side)
                l0 = li + 1
        main.wait_stream(side)

    def _capture(self) -> None:
        # capture mutates device token counters when kernels run? No: capture
        # only records.  Warm the kernels (function attributes) outside capture
        # on a throw-away copy of nothing: attributes are set at first launch,
        # which is allowed during capture.
        for select in (True, False):
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream(device=self.dev)
            s.wait_stream(torch.cuda.current_stream(self.dev))
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    self._launch_step(select)
            torch.cuda.current_stream(self.dev).wait_stream(s)
            self.graphs[select] = g

    # -- stepping ---------------------------------------------------------------
    def step(self) -> torch.Tensor:
        """Run one decode step for every layer on the current contents of
        self.q / self.k / self.v; returns self.out (device)."""
        if self.steps_done >= self.max_steps:
            raise RuntimeError("DecodeGraph capacity exhausted; build a new one")
        cfg = self.cfg
        step = self.engines[0].decode_steps
        if step != self._next_step:  # the engines were stepped outside this runner: rescan their states
            self._valid = None
        self._next_step = step + 1
        if self._valid is None:  # steps [lo, hi) every stream's selection state covers
            lo, hi = -1, -1
            states = [e.selection_states.get(kv) for e in self.engines for kv in e.cache.dense_pool
                      if e._row_mask_host[kv]]
            if all(st is not None and st.budget_tokens == cfg.budget_tokens and
                   st.reuse_interval == cfg.reuse_interval for st in states):
                lo = max((st.chunk_start_step for st in states), default=0)
                hi = min((st.chunk_start_step + cfg.reuse_interval for st in states), default=1 << 62)
            self._valid = (lo, hi)
        select = not (self._valid[0] <= step < self._valid[1])
        self.graphs[select].replay()
        # host bookkeeping (overlaps the replay): mirrors Engine.decode_step
        n_tok = self.start_tokens + self.steps_done
        n_pages = -(-n_tok // cfg.physical_page)
        if select:
            from .selector import SelectionState
            self._valid = (step, step + cfg.reuse_interval)
            pg = cfg.physical_page
            sizes = [selection_size(-(-(t + self.steps_done) // pg), self.k_pages) for t in self.start_per_stream]
        for e, pool in zip(self.engines, self.pools):
            if select:
                states = e.selection_states
                for kv in e.cache.dense_pool:
                    if e._row_mask_host[kv]:
                        st = states.get(kv)
                        if isinstance(st, SelectionState) and isinstance(st.selected_pages, _Sized):
                            st.selected_pages._n = sizes[kv]  # this runner's own state: refresh in place
                            st.chunk_start_step = step
                            st.reuse_interval, st.budget_tokens = cfg.reuse_interval, cfg.budget_tokens
                        else:
                            states[kv] = SelectionState(_Sized(sizes[kv]), step, cfg.reuse_interval,
                                                        cfg.budget_tokens)
                        e.ledger.record_selector(kv)
            if self.record_ledger:
                for hh, prof in enumerate(e.profiles):
                    kv = hh // self.g
                    if prof.role == RETRIEVAL:
                        vis = len(e.selection_states[kv].selected_pages)
                    else:
                        vis = sum(b - a for a, b in lambda_segments(n_pages, prof.sink_blocks, prof.local_blocks,
                                                                     n_pages - 1))
                    e.ledger.record_tiles(DECODE, hh, vis, n_pages)
            pool.tokens_host[:] = [t + 1 for t in pool.tokens_host]
            e.decode_steps += 1
        self.steps_done += 1
        return self.out


class _Sized(list):
    """Placeholder selection list of known length (contents stay on device)."""

    def __init__(self, n: int):
        super().__init__()
        self._n = n

    def __len__(self) -> int:
        return self._n
