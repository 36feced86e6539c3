"""Prefill / decode orchestration on the B200.

Same API as the reference ``sparsekv.engine`` (engine.py:30-310): one
``Engine`` is one attention layer of one sequence.  Host work is integer
bookkeeping only (roles, schedules -> work lists, reuse windows, ledger);
every tensor operation is a kernel of the C-ABI library:

  prefill      K4 block-sparse tcgen05 attention on raw K/V, then K1 bulk
               append into the two-way device pool
  load_context K1 bulk append
  decode_step  K2 selection (only on reuse-window starts) -> K3 split-KV
               decode with the new token in-register and the append fused
               into the same launch

Nothing synchronises with the host unless the caller passes numpy arrays
(then the output is copied back) or reads ``DecodeResult.index_tables``
(lazily materialised).
"""

from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import asdict, dataclass, field
from pathlib import Path
from typing import Sequence

import numpy as np
import torch

from . import _device, _lib
from .attn import (Workload, check_finite_device, diagonal_tile, kv_tile_count, plan_from_segments, plan_generic,
                   query_tile_count, run_prefill, run_prefill_paged)
from .cache import TwoWayCache
from .heads import RETRIEVAL, HeadProfile, lambda_segments
from .ledger import CostLedger
from .selector import SelectionState, pinned_pages, select_streams, selection_size

PREFILL = "prefill"
DECODE = "decode"


@dataclass
class EngineConfig:
    """engine.py:30-83 -- field for field."""

    physical_page: int = 64
    logical_page: int = 16
    quant_bits: int | None = 4
    budget_tokens: int = 4096
    reuse_interval: int = 4
    sink_blocks: int = 1
    local_blocks: int = 2
    target_sparsity: float = 0.5
    tile_q_prefill: int = 64
    seed: int = 0

    def __post_init__(self):
        if self.quant_bits == 0:
            self.quant_bits = None
        if self.physical_page < 1 or self.logical_page < 1:
            raise ValueError("page sizes must be >= 1")
        if self.physical_page % self.logical_page != 0:
            raise ValueError(f"logical page {self.logical_page} must divide physical page {self.physical_page}")
        if self.quant_bits is not None and not 2 <= self.quant_bits <= 8:
            raise ValueError("quant_bits must be 0/null or in [2, 8]")
        if self.budget_tokens < self.physical_page:
            raise ValueError(f"budget_tokens {self.budget_tokens} is below one physical page "
                             f"({self.physical_page} tokens)")
        if self.reuse_interval < 1:
            raise ValueError("reuse_interval must be >= 1")
        if self.sink_blocks < 1 or self.local_blocks < 1:
            raise ValueError("sink_blocks and local_blocks must be >= 1")
        if not 0.0 <= self.target_sparsity < 1.0:
            raise ValueError("target_sparsity must be in [0, 1)")
        if self.tile_q_prefill < 1:
            raise ValueError("tile_q_prefill must be >= 1")

    def to_dict(self) -> dict:
        return asdict(self)

    @classmethod
    def from_dict(cls, data: dict) -> "EngineConfig":
        unknown = set(data) - set(cls.__dataclass_fields__)
        if unknown:
            raise ValueError(f"unknown config keys: {sorted(unknown)}")
        return cls(**data)

    @classmethod
    def from_json(cls, path) -> "EngineConfig":
        with open(path) as fp:
            return cls.from_dict(json.load(fp))


@dataclass(frozen=True)
class IndexTable:
    """engine.py:86-98."""

    head: int
    positions: tuple

    def __post_init__(self):
        if any(b <= a for a, b in zip(self.positions, self.positions[1:])):
            raise ValueError("index table positions must be strictly increasing")

    def __len__(self) -> int:
        return len(self.positions)


class DevicePageList(Sequence):
    """A selection living on the device (row `row` of `sel`, `count[row]`
    entries); materialised into Python ints on first access."""

    def __init__(self, sel: torch.Tensor, count: torch.Tensor, row: int, size: int):
        self._sel, self._count, self._row, self._size = sel, count, row, size
        self._host = None

    def _mat(self) -> list:
        if self._host is None:
            self._host = self._sel[self._row, :self._size].cpu().tolist()
        return self._host

    def __len__(self) -> int:
        return self._size

    def __getitem__(self, i):
        return self._mat()[i]

    def __iter__(self):
        return iter(self._mat())

    def __eq__(self, other):
        return list(self) == list(other)

    def __repr__(self) -> str:
        return f"DevicePageList({self._mat()!r})"


class _LazyTables(Sequence):
    def __init__(self, make):
        self._make, self._tables = make, None

    def _mat(self):
        if self._tables is None:
            self._tables = self._make()
        return self._tables

    def __len__(self):
        return len(self._mat())

    def __getitem__(self, i):
        return self._mat()[i]


@dataclass
class DecodeResult:
    """engine.py:101-105."""

    output: object
    index_tables: Sequence
    invoked: dict = field(default_factory=dict)


class Engine:
    """engine.py:108-286 -- one layer of one sequence, device resident."""

    def __init__(self, config: EngineConfig, profiles: list, *, dtype: torch.dtype = _device.DEFAULT_DTYPE,
                 device=None, capacity_tokens: int = 0, paged_history: bool | None = None):
        self.config = config
        # chunked prefill over KV4 history: True = K4 reads pages through the page table,
        # False = K1b gathers the history into a dense buffer first (faster),
        # None = gather unless the dense buffer would not fit in half the free HBM
        self.paged_history = paged_history
        self.profiles = profiles
        self.cache: TwoWayCache | None = None
        self.ledger = CostLedger()
        self.selection_states: dict = {}
        self.decode_steps = 0
        self._group_size: int | None = None
        self._dtype, self._device_arg, self._capacity = dtype, device, capacity_tokens
        self._plans: dict = {}
        self._sel = None

    # -- helpers ----------------------------------------------------------------
    def _group_heads(self, kv_head: int) -> list:
        n = self._group_size
        return list(range(kv_head * n, (kv_head + 1) * n))

    def _dense_kv_heads(self, num_kv_heads: int) -> set:
        """engine.py:126-132."""
        return {kv for kv in range(num_kv_heads)
                if any(self.profiles[h].role == RETRIEVAL for h in self._group_heads(kv))}

    @property
    def device(self) -> torch.device:
        return _device.device_of(self._device_arg)

    def _new_cache(self, num_kv_heads: int, head_dim: int, tokens: int) -> None:
        cfg = self.config
        dense = self._dense_kv_heads(num_kv_heads)
        old = self.cache.pool if self.cache is not None else None
        self.cache = TwoWayCache(cfg.physical_page, cfg.logical_page, cfg.quant_bits, dense,
                                 set(range(num_kv_heads)) - dense, cfg.sink_blocks, cfg.local_blocks,
                                 dtype=self._dtype, device=self.device,
                                 capacity_tokens=max(self._capacity, tokens + 1))
        # A fresh cache (engine.py:146-150) recycles the previous device pool when
        # the geometry matches: emptied by a device-side reset, so a re-prefill
        # issues no host->device copies on the compute stream (they would queue
        # behind bulk uploads on the copy engine, see pipeline.py).
        if old is not None and old.matches(self.cache.pool_kinds(), head_dim, cfg.physical_page, cfg.logical_page,
                                           cfg.quant_bits, cfg.sink_blocks, cfg.local_blocks, self._dtype):
            old.reset()
            old.reserve(tokens + 1)
            self.cache.adopt_pool(old)
        else:
            self.cache.ensure_pool(head_dim)
        masks = []
        for kv in range(num_kv_heads):
            mk = 0
            for r, h in enumerate(self._group_heads(kv)):
                if self.profiles[h].role == RETRIEVAL:
                    mk |= 1 << r
            masks.append(mk)
        if getattr(self, "_row_mask_host", None) != masks:
            self._row_mask = _device.h2d(np.array(masks, np.int32), self.device)
        self._row_mask_host = masks
        # per-row streaming windows for K3, only when a profile differs from the pool's
        wins = [[self._window_of(h) for h in self._group_heads(kv)] for kv in range(num_kv_heads)]
        pool_win = cfg.sink_blocks | (cfg.local_blocks << 16)
        if all(w == pool_win for row in wins for w in row):
            self._row_window = None
        else:
            self._row_window = _device.h2d(np.array(wins, np.uint32), self.device)
        self._sel = None
        self.selection_states = {}

    def _window_of(self, h: int) -> int:
        """sink | local << 16 of streaming head h (retrieval rows: the pool's)."""
        p, cfg = self.profiles[h], self.config
        if p.role == RETRIEVAL:
            return cfg.sink_blocks | (cfg.local_blocks << 16)
        return p.sink_blocks | (p.local_blocks << 16)

    def _check_windows(self, n_pages: int) -> None:
        """A streaming-pool KV head keeps only the pool's sink + local pages
        (cache.py:253-261); a profile asking for more reads an evicted page,
        which the reference refuses (page_at -> KeyError)."""
        cfg, g = self.config, self._group_size
        for kv in self.cache.streaming_pool:
            for h in self._group_heads(kv):
                p = self.profiles[h]
                want = {t for a, b in lambda_segments(n_pages, p.sink_blocks, p.local_blocks, n_pages - 1)
                        for t in range(a, b)}
                live = set(self.cache.pool.live_indices(self.cache.stream_of[kv]))
                missing = sorted(want - live)
                if missing:
                    raise KeyError(f"page index {missing[0]} is not resident: head {h}'s window "
                                   f"({p.sink_blocks}, {p.local_blocks}) reaches evicted pages of KV head {kv}")

    def _plan(self, n: int, s: int):
        cfg = self.config
        key = (n, s, cfg.tile_q_prefill, cfg.physical_page,
               tuple((p.role, p.sink_blocks, p.local_blocks) for p in self.profiles))
        plan = self._plans.get(key)
        if plan is not None:
            return plan
        tq, tk = cfg.tile_q_prefill, cfg.physical_page
        n_tiles = kv_tile_count(s, tk)

        def head_segments(h, qt):
            dg = diagonal_tile(qt, tq, tk, n, s)
            p = self.profiles[h]
            if p.role == RETRIEVAL:
                return ((0, dg + 1),)
            return lambda_segments(n_tiles, p.sink_blocks, p.local_blocks, dg)

        if tq == 64 and tk == 64:
            plan = plan_from_segments(head_segments, len(self.profiles), n, s)
        else:
            sched = {(h, qt): [t for a, b in head_segments(h, qt) for t in range(a, b)]
                     for h in range(len(self.profiles)) for qt in range(query_tile_count(n, tq))}
            plan = plan_generic(sched, len(self.profiles), n, s, tq, tk)
        self._plans[key] = plan
        return plan

    # -- prefill ----------------------------------------------------------------
    def prefill(self, w: Workload):
        """engine.py:136-173: K4 over the static schedules, then K1 bulk append."""
        if len(self.profiles) != w.num_heads:
            raise ValueError(f"{len(self.profiles)} profiles for {w.num_heads} heads")
        self._group_size = w.group_size
        n, s = w.num_queries, w.num_history
        dev = self.device
        dp = _device.padded_dim(w.head_dim)
        q = _device.to_device(w.q, self._dtype, dev, dp)
        k = _device.to_device(w.k, self._dtype, dev, dp)
        v = _device.to_device(w.v, self._dtype, dev, dp)
        check_finite_device(w, q, k, v)
        out = self.prefill_device(q, k, v, w.head_dim)
        np_dt = None if _device.is_torch(w.q) else np.asarray(w.q).dtype
        return _device.to_output(out[..., :w.head_dim], w.q, np_dt)

    def prefill_device(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, head_dim: int) -> torch.Tensor:
        """Device fast path: q [N,H,Dp], k/v [S,Hkv,Dp] already padded, dtype-cast."""
        n, h, dp = q.shape
        s, h_kv, _ = k.shape
        if h % h_kv:
            raise ValueError(f"query head count {h} is not a multiple of KV head count {h_kv}")
        self._group_size = h // h_kv
        self._new_cache(h_kv, head_dim, s)
        plan = self._plan(n, s)
        out = run_prefill(q, k, v, plan, 1.0 / math.sqrt(head_dim))
        for hh in range(h):
            self.ledger.record_tiles(PREFILL, hh, int(plan.visited[hh]), int(plan.total[hh]))
        self.cache._user_dim = head_dim
        self.cache.append_all(k, v)
        return out

    def prefill_chunk(self, w: Workload):
        """Continued (chunked) prefill -- an extension, the reference has no such
        entry point.  ``w.q`` [n, H, D] are the chunk's queries at positions
        S0..S0+n-1 and ``w.k``/``w.v`` [n, Hkv, D] its own keys/values; the
        chunk attends the cached history (dequantised exactly as the decode
        path reads it, engine.py:250-262) plus its own raw K/V under the static
        prefill schedules of an (n, S0+n) workload (engine.py:152-165), then is
        appended to the cache.  On an empty engine this is ``prefill``."""
        if self.cache is None or self.cache.pool is None or self.cache.num_tokens == 0:
            return self.prefill(w)
        if len(self.profiles) != w.num_heads:
            raise ValueError(f"{len(self.profiles)} profiles for {w.num_heads} heads")
        pool = self.cache.pool
        if w.head_dim != self.cache._user_dim or w.k.shape[1] != pool.n_streams:
            raise ValueError("chunk shapes do not match the cached history")
        dp = pool.Dp
        q = _device.to_device(w.q, self._dtype, self.device, dp)
        k = _device.to_device(w.k, self._dtype, self.device, dp)
        v = _device.to_device(w.v, self._dtype, self.device, dp)
        check_finite_device(w, q, k, v)
        out = self.prefill_chunk_device(q, k, v, w.head_dim)
        np_dt = None if _device.is_torch(w.q) else np.asarray(w.q).dtype
        return _device.to_output(out[..., :w.head_dim], w.q, np_dt)

    def prefill_chunk_device(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, head_dim: int) -> torch.Tensor:
        """Device fast path of prefill_chunk: q [n,H,Dp], k/v [n,Hkv,Dp] padded, pool dtype."""
        if self.cache is None or self.cache.pool is None or self.cache.num_tokens == 0:
            return self.prefill_device(q, k, v, head_dim)
        cfg = self.config
        pool = self.cache.pool
        n, h, dp = q.shape
        if h != len(self.profiles) or h != self._group_size * pool.n_streams or tuple(k.shape) != (n, pool.n_streams, dp):
            raise ValueError("chunk shapes do not match the cached history")
        for p in self.profiles:  # streaming heads may only reach pages their ring keeps
            if p.role != RETRIEVAL and (p.sink_blocks > cfg.sink_blocks or p.local_blocks > cfg.local_blocks):
                raise ValueError(f"head {p.head}: window ({p.sink_blocks}, {p.local_blocks}) exceeds the "
                                 f"streaming pool's ({cfg.sink_blocks}, {cfg.local_blocks}); evicted pages "
                                 "cannot be attended")
        s0 = self.cache.num_tokens
        plan = self._plan(n, s0 + n)
        if 1 <= pool.bits <= 4 and pool.P in (32, 64) and self._use_paged(pool, s0 + n, dp):
            # K4 reads the KV4 history through the page table (no history buffer)
            out = run_prefill_paged(pool, s0, q, k.contiguous(), v.contiguous(), plan, 1.0 / math.sqrt(head_dim))
        else:  # KV8 / raw pages: K1b expands the history once, K4 streams it with TMA
            kh, vh = pool.gather(extra_tokens=n)
            kh[s0:] = k
            vh[s0:] = v
            out = run_prefill(q, kh, vh, plan, 1.0 / math.sqrt(head_dim))
            del kh, vh
        for hh in range(h):
            self.ledger.record_tiles(PREFILL, hh, int(plan.visited[hh]), int(plan.total[hh]))
        self.cache.append_all(k, v)
        return out

    def _use_paged(self, pool, tokens: int, dp: int) -> bool:
        if self.paged_history is not None:
            return bool(self.paged_history)
        need = 2 * tokens * pool.n_streams * dp * torch.empty((), dtype=self._dtype).element_size()
        free, _ = torch.cuda.mem_get_info(self.device)
        return need > free // 2

    def load_context(self, k_history, v_history) -> None:
        """engine.py:175-204: K1 bulk append, no attention."""
        shape_k, shape_v = tuple(np.shape(k_history)), tuple(np.shape(v_history))
        if len(shape_k) != 3 or shape_k != shape_v:
            raise ValueError("history must be [tokens, num_kv_heads, head_dim]")
        h_kv = shape_k[1]
        if len(self.profiles) % h_kv != 0:
            raise ValueError(f"{len(self.profiles)} heads not divisible by {h_kv} KV heads")
        self._group_size = len(self.profiles) // h_kv
        dp = _device.padded_dim(shape_k[2])
        k = _device.to_device(k_history, self._dtype, self.device, dp)
        v = _device.to_device(v_history, self._dtype, self.device, dp)
        self._new_cache(h_kv, shape_k[2], shape_k[0])
        self.cache._user_dim = shape_k[2]
        self.cache.append_all(k, v)

    # -- decode -------------------------------------------------------------------
    def decode_step(self, q_new, k_new, v_new) -> DecodeResult:
        """engine.py:208-286."""
        if self.cache is None or self.cache.pool is None or self.cache.num_tokens == 0:
            raise ValueError("decode_step requires a non-empty cache")
        h, d = tuple(np.shape(q_new))
        h_kv = np.shape(k_new)[0]
        if h != len(self.profiles) or h % h_kv != 0:
            raise ValueError("decode head shapes do not match the profiles")
        self._group_size = h // h_kv
        pool = self.cache.pool
        dp = pool.Dp
        q = _device.to_device(q_new, self._dtype, self.device, dp)
        kn = _device.to_device(k_new, self._dtype, self.device, dp)
        vn = _device.to_device(v_new, self._dtype, self.device, dp)
        out = self.decode_device(q, kn, vn, d)
        np_dt = None if _device.is_torch(q_new) else np.asarray(q_new).dtype
        return DecodeResult(_device.to_output(out[:, :d], q_new, np_dt), self._last_tables, self._last_invoked)

    def row_window_ptr(self):
        w = getattr(self, "_row_window", None)
        return None if w is None else w.data_ptr()

    def decode_device(self, q: torch.Tensor, kn: torch.Tensor, vn: torch.Tensor, head_dim: int) -> torch.Tensor:
        """Device fast path: q [H,Dp], kn/vn [Hkv,Dp] in the pool dtype."""
        cfg = self.config
        pool = self.cache.pool
        g = self._group_size
        h_kv = pool.n_streams
        n_tok = self.cache.num_tokens
        n_pages = -(-n_tok // cfg.physical_page)
        k_pages = -(-cfg.budget_tokens // cfg.physical_page)
        step = self.decode_steps
        dev = self.device
        # -- selection (K2) on reuse-window starts ----------------------------------
        invoked = {}
        need = []
        for kv in sorted(self.cache.dense_pool):
            if not self._row_mask_host[kv]:
                continue
            st = self.selection_states.get(kv)
            run = not (st is not None and st.valid_for(step, cfg.budget_tokens, cfg.reuse_interval))
            invoked[kv] = run
            if run:
                need.append(kv)
        if need:
            width = max(4, k_pages)
            active = [kv for kv in range(h_kv) if self._row_mask_host[kv]]
            if self._sel is not None and len(need) < len(active) and self._sel[0].shape[1] == width:
                # partial invocation: keep the other streams' selections (copy: the
                # previous tensors back DevicePageLists that must stay immutable)
                sel, cnt = self._sel[0].clone(), self._sel[1].clone()
                inv = _device.h2d(np.array([1 if kv in need else 0 for kv in range(h_kv)], np.uint8), dev)
            else:
                sel = torch.empty((h_kv, width), dtype=torch.int32, device=dev)
                cnt = torch.zeros(h_kv, dtype=torch.int32, device=dev)
                inv = None
            select_streams(pool, q, g * pool.Dp, pool.Dp, g, self._row_mask, k_pages, sel, cnt, invoke=inv,
                           max_pages_hint=max(1, n_pages))
            self._sel = (sel, cnt)
            size = selection_size(n_pages, k_pages)
            for kv in need:
                self.selection_states[kv] = SelectionState(DevicePageList(sel, cnt, kv, size), step,
                                                           cfg.reuse_interval, cfg.budget_tokens)
                self.ledger.record_selector(kv)
        # -- attention + fused append (K3) -----------------------------------------
        pool.reserve(n_tok + 1)
        sel, cnt = self._sel if self._sel is not None else (
            torch.zeros((h_kv, 4), dtype=torch.int32, device=dev), torch.zeros(h_kv, dtype=torch.int32, device=dev))
        if self._row_window is not None:
            self._check_windows(n_pages)
        out = torch.empty((h_kv * g, pool.Dp), dtype=self._dtype, device=dev)
        abi = pool.abi()
        dws = pool.decode_workspace(g)
        rc = _lib.load().sk_decode_attn(
            C.byref(abi), h_kv, g, q.data_ptr(), g * pool.Dp, pool.Dp, kn.data_ptr(), vn.data_ptr(), pool.Dp,
            self._row_mask.data_ptr(), self.row_window_ptr(), sel.data_ptr(), cnt.data_ptr(), sel.shape[1],
            pool.tokens.data_ptr(), C.c_float(1.0 / math.sqrt(head_dim)), out.data_ptr(), g * pool.Dp, pool.Dp,
            _device.sk_dtype(self._dtype), 1, dws.data_ptr(), dws.numel(), _device.stream_ptr(dev))
        _lib.check(rc)
        for s in range(h_kv):
            pool.tokens_host[s] += 1
        # -- ledger + lazily materialised index tables ----------------------------
        tables_spec = []
        for hh, prof in enumerate(self.profiles):
            kv = hh // g
            if prof.role == RETRIEVAL:
                st = self.selection_states[kv]
                tables_spec.append((hh, st.selected_pages))
                self.ledger.record_tiles(DECODE, hh, len(st.selected_pages), n_pages)
            else:
                segs = lambda_segments(n_pages, prof.sink_blocks, prof.local_blocks, n_pages - 1)
                tiles = tuple(t for a, b in segs for t in range(a, b))
                tables_spec.append((hh, tiles))
                self.ledger.record_tiles(DECODE, hh, len(tiles), n_pages)
        self._last_tables = _LazyTables(lambda spec=tables_spec: [IndexTable(hh, tuple(int(x) for x in pos))
                                                                 for hh, pos in spec])
        self._last_invoked = invoked
        self.decode_steps += 1
        return out


def cost_report(ledger: CostLedger) -> dict:
    """engine.py:289-310."""
    stages = {}
    for stage in ledger.stages():
        stages[stage] = {"visited_tiles": ledger.visited(stage), "total_tiles": ledger.total(stage),
                         "skip_fraction": ledger.skip_fraction(stage), "speedup": ledger.speedup(stage)}
    return {"stages": stages,
            "selector_invocations": {"total": ledger.total_selector_invocations,
                                     "per_kv_head": {str(kv): c for kv, c in
                                                     sorted(ledger.selector_invocations.items())}}}
