"""Batched decode over many sequences (BASELINE cfg4; an extension outside the
reference API).

The reference engine is "one instance per sequence" with cross-sequence
parallelism left to the caller.  On the B200 one sequence's
decode step is far too small to fill the GPU, so a serving step batches
sequences: `BatchedLayer` keeps ONE device pool per layer whose streams are
(sequence, KV head) pairs -- stream b*Hkv + kv, each with its own page-table
row ("per-sequence page tables") and token count -- so K2, K3 and K1 each run
once per layer for the whole batch.  It exposes the attributes
`decode_graph.DecodeGraph` drives, so the same multi-layer CUDA graph runs
the batch.  Per-sequence semantics (selection reuse, streaming windows,
append after attention) are exactly those of `Engine.decode_step`; the
parity test checks every sequence against its own `Engine`.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device, _lib
from .cache import DevicePool
from .engine import EngineConfig
from .heads import RETRIEVAL
from .ledger import CostLedger


class _StreamsView:
    def __init__(self, pool: DevicePool, dense_streams):
        self.pool = pool
        self.dense_pool = {s: None for s in dense_streams}


class BatchedLayer:
    """One attention layer of `batch` sequences in one device pool."""

    def __init__(self, config: EngineConfig, profiles: list, batch: int, num_kv_heads: int, head_dim: int, *,
                 dtype: torch.dtype = _device.DEFAULT_DTYPE, device=None, capacity_tokens: int = 0):
        if len(profiles) % num_kv_heads:
            raise ValueError(f"{len(profiles)} heads not divisible by {num_kv_heads} KV heads")
        if batch < 1:
            raise ValueError("batch must be >= 1")
        self.config, self.profiles, self.batch = config, profiles, batch
        self.h_kv = num_kv_heads
        self._group_size = len(profiles) // num_kv_heads
        self.device = _device.device_of(device)
        g = self._group_size
        masks = []
        for kv in range(num_kv_heads):
            mk = 0
            for r in range(g):
                if profiles[kv * g + r].role == RETRIEVAL:
                    mk |= 1 << r
            masks.append(mk)
        kinds = [_lib.SK_KIND_DENSE if masks[kv] else _lib.SK_KIND_STREAMING
                 for _ in range(batch) for kv in range(num_kv_heads)]
        self.pool = DevicePool(kinds, head_dim, config.physical_page, config.logical_page, config.quant_bits,
                               config.sink_blocks, config.local_blocks, dtype, self.device, capacity_tokens)
        self._row_mask_host = masks * batch
        self._row_mask = _device.h2d(torch.tensor(self._row_mask_host, dtype=torch.int32).numpy(), self.device)
        pool_win = config.sink_blocks | (config.local_blocks << 16)
        wins = [pool_win if p.role == RETRIEVAL else (p.sink_blocks | (p.local_blocks << 16)) for p in profiles]
        if any(kinds[kv] == _lib.SK_KIND_STREAMING and any(w != pool_win for w in wins[kv * g:(kv + 1) * g])
               for kv in range(num_kv_heads)):
            raise KeyError("a streaming head's window differs from the streaming pool's (evicted pages)")
        self._row_window = None if all(w == pool_win for w in wins) else \
            _device.h2d(np.array(wins * batch, np.uint32), self.device)
        self.cache = _StreamsView(self.pool, [s for s, k in enumerate(kinds) if k == _lib.SK_KIND_DENSE])
        self.selection_states: dict = {}
        self.ledger = CostLedger()
        self.decode_steps = 0

    def row_window_ptr(self):
        return None if self._row_window is None else self._row_window.data_ptr()

    def load_context(self, seq: int, k: torch.Tensor, v: torch.Tensor) -> None:
        """K1 bulk append of one sequence's history (device [S, Hkv, Dp], pool dtype)."""
        if not 0 <= seq < self.batch:
            raise ValueError(f"sequence {seq} outside the batch of {self.batch}")
        m, h_kv, dp = k.shape
        if h_kv != self.h_kv or dp != self.pool.Dp:
            raise ValueError(f"history shape {tuple(k.shape)} does not match ({self.h_kv}, {self.pool.Dp})")
        self.pool.append(k, v, dp, h_kv * dp, m, first_stream=seq * self.h_kv, n_streams=self.h_kv)
