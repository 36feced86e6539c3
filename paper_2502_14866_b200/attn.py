"""Attention: workload validation, tile geometry, online softmax and the
block-sparse prefill entry point.

API mirrors the reference ``sparsekv.attn`` (attn.py:23-324).  The hot
path, :func:`blockwise_attention`, validates the schedules on the host,
compiles them into 256-row work items over 64-key block segments and runs
the tcgen05 prefill kernel (csrc/prefill.cu) -- there is no CPU fallback.
Inputs may be numpy arrays or torch tensors; they are computed in the
device dtype (fp16 by default, bf16 optional) and returned in the caller's
flavour (numpy in -> numpy out in the input dtype).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Iterable, Mapping, Sequence

import numpy as np
import torch

from . import _device, _lib
from .ledger import CostLedger

NEG_INF = -np.inf


@dataclass
class Workload:
    """attn.py:23-87 -- q [N, H, D], k/v [S, Hkv, D] (numpy or torch)."""

    q: object
    k: object
    v: object

    def __post_init__(self) -> None:
        q, k, v = self.q, self.k, self.v
        conv = (lambda t: t) if _device.is_torch(q) else np.asarray
        q, k, v = conv(q), conv(k), conv(v)
        if q.ndim != 3 or k.ndim != 3 or v.ndim != 3:
            raise ValueError("q, k, v must be rank-3 [tokens, heads, dim]")
        if tuple(k.shape) != tuple(v.shape):
            raise ValueError(f"k and v shapes differ: {tuple(k.shape)} vs {tuple(v.shape)}")
        if q.shape[2] != k.shape[2]:
            raise ValueError("head_dim mismatch between q and k")
        if min(q.shape) < 1 or min(k.shape) < 1:
            raise ValueError("all tensor dimensions must be positive")
        if q.shape[1] % k.shape[1] != 0:
            raise ValueError(f"query head count {q.shape[1]} is not a multiple of KV head count {k.shape[1]}")
        for name, t in (("q", q), ("k", k), ("v", v)):
            if _device.is_torch(t) and not t.is_cuda:
                continue  # host torch tensors are checked on the device after upload (Engine / blockwise)
            finite = bool(_device.all_finite(t)) if _device.is_torch(t) else bool(np.isfinite(t).all())
            if not finite:
                raise ValueError(f"non-finite values in {name}")
        self.q, self.k, self.v = q, k, v

    num_queries = property(lambda self: self.q.shape[0])
    num_history = property(lambda self: self.k.shape[0])
    num_heads = property(lambda self: self.q.shape[1])
    num_kv_heads = property(lambda self: self.k.shape[1])
    head_dim = property(lambda self: self.q.shape[2])
    group_size = property(lambda self: self.q.shape[1] // self.k.shape[1])

    def astype(self, dtype) -> "Workload":
        if _device.is_torch(self.q):
            return Workload(self.q.to(dtype), self.k.to(dtype), self.v.to(dtype))
        return Workload(self.q.astype(dtype), self.k.astype(dtype), self.v.astype(dtype))


def gqa_map(head: int, group_size: int) -> int:
    """attn.py:90-96."""
    if head < 0:
        raise IndexError(f"query head index {head} out of range")
    if group_size < 1:
        raise ValueError(f"group size must be >= 1, got {group_size}")
    return head // group_size


def kv_tile_count(num_history: int, tile_k: int) -> int:
    return -(-num_history // tile_k)


def query_tile_count(num_queries: int, tile_q: int) -> int:
    return -(-num_queries // tile_q)


def diagonal_tile(query_tile: int, tile_q: int, tile_k: int, num_queries: int, num_history: int) -> int:
    """attn.py:111-115."""
    q_last = min((query_tile + 1) * tile_q, num_queries) - 1
    return (num_history - num_queries + q_last) // tile_k


def full_causal_schedule(query_tile: int, tile_q: int, tile_k: int, num_queries: int, num_history: int) -> range:
    return range(diagonal_tile(query_tile, tile_q, tile_k, num_queries, num_history) + 1)


# -- reference-style utilities (not the hot path) ------------------------------


def reference_attention(w: Workload, causal: bool = True):
    """attn.py:128-162 -- dense fp64 softmax oracle (torch fp64 on the inputs' device)."""
    n, s = w.num_queries, w.num_history
    if causal and s < n:
        raise ValueError(f"causal attention needs history >= queries, got S={s}, N={n}")
    as_t = (lambda t: t.double()) if _device.is_torch(w.q) else (lambda t: torch.from_numpy(np.asarray(t, np.float64)))
    q, k, v = as_t(w.q), as_t(w.k), as_t(w.v)
    kk = k.repeat_interleave(w.group_size, dim=1)
    vv = v.repeat_interleave(w.group_size, dim=1)
    sc = torch.einsum("nhd,shd->hns", q, kk) / math.sqrt(w.head_dim)
    if causal:
        hide = torch.arange(s, device=sc.device)[None, :] > (torch.arange(n, device=sc.device)[:, None] + s - n)
        sc = sc.masked_fill(hide[None], float("-inf"))
    out = torch.einsum("hns,shd->nhd", torch.softmax(sc, dim=-1), vv)
    return out if _device.is_torch(w.q) else out.numpy()


@dataclass
class SoftmaxState:
    """attn.py:168-188 -- running max / denominator / output."""

    running_max: np.ndarray
    running_denominator: np.ndarray
    running_output: np.ndarray

    @classmethod
    def initial(cls, rows: int, dim: int, dtype=np.float64) -> "SoftmaxState":
        return cls(np.full(rows, NEG_INF, dtype=dtype), np.zeros(rows, dtype=dtype), np.zeros((rows, dim), dtype=dtype))

    def finalize(self) -> np.ndarray:
        if np.any(self.running_denominator <= 0):
            raise ValueError("row with no attended positions (denominator is 0)")
        return self.running_output / self.running_denominator[:, None]


def merge_block(state: SoftmaxState, scores, values) -> SoftmaxState:
    """attn.py:191-229 -- one online-softmax step (host utility)."""
    scores = np.asarray(scores)
    if scores.ndim == 1:
        scores = scores[None, :]
    values = np.asarray(values)
    if np.any(np.isposinf(scores)) or np.any(np.isnan(scores)):
        raise ValueError("scores must be finite or -inf")
    if not np.isfinite(values).all():
        raise ValueError("values must be finite")
    dt = state.running_max.dtype
    m_old = state.running_max
    m_new = np.maximum(m_old, scores.max(axis=1))
    shift = np.where(m_new > NEG_INF, m_new, 0.0).astype(dt)
    probs = np.exp(scores - shift[:, None])
    alpha = np.where(m_old > NEG_INF, np.exp(m_old - shift), 0.0).astype(dt)
    return SoftmaxState(m_new, alpha * state.running_denominator + probs.sum(axis=1),
                        alpha[:, None] * state.running_output + probs @ values)


# -- prefill plan: schedules -> 256-row work items over 64-key segments --------


def _segments_of(tiles: Sequence[int]) -> tuple:
    out = []
    for t in tiles:
        if out and out[-1][1] == t:
            out[-1][1] = t + 1
        else:
            out.append([t, t + 1])
    return tuple((a, b) for a, b in out)


def _inside(segs, x) -> bool:
    return any(a <= x < b for a, b in segs)


ITEM_ROWS = 256  # query rows per K4 work item: two 128-row tcgen05 tiles = four reference q-tiles
F_CAUSAL, F_MASKS = 1 << 4, 1 << 5  # segment flags above the four per-quarter bits


def _item_segments(quarters, row0: int, n: int, s: int) -> list:
    """Union of the four 64-row quarters' tile segments with per-quarter
    and causal flags (native 64x64 tiling; tiles == 64-key blocks)."""
    cb = max(0, (row0 + s - n - 63) // 64 + 1)  # first block whose last column passes row0's position
    pts = {cb}
    for segs in quarters:
        for a, b in segs or ():
            pts.update((a, b))
    pts = sorted(pts)
    out = []
    for x, y in zip(pts, pts[1:]):
        fl = 0
        for qi, segs in enumerate(quarters):
            if segs and _inside(segs, x):
                fl |= 1 << qi
        if not fl:
            continue
        if x >= cb:
            fl |= F_CAUSAL
        if out and out[-1][0] + out[-1][1] == x and out[-1][2] == fl:
            out[-1][1] += y - x
        else:
            out.append([x, y - x, fl])
    return out


class PrefillPlan:
    """Device work list for one (schedules, geometry): items sorted heaviest
    first, segments, optional explicit row masks, and the ledger counts."""

    def __init__(self, items: np.ndarray, segs: np.ndarray, masks, visited: np.ndarray, total: np.ndarray):
        self.items_np, self.segs_np, self.masks_np = items, segs, masks
        self.visited, self.total = visited, total
        self._dev = {}

    def device_arrays(self, device):
        key = str(device)
        if key not in self._dev:
            it = _device.h2d(self.items_np, device)
            sg = _device.h2d(self.segs_np.view(np.int32), device)
            mk = _device.h2d(self.masks_np.view(np.int64), device) if self.masks_np is not None else None
            self._dev[key] = (it, sg, mk)
        return self._dev[key]

    @property
    def n_items(self) -> int:
        return self.items_np.shape[0]


def _finish_plan(items, segs, masks, visited, total) -> PrefillPlan:
    cost = np.array([sum(segs[i][1] for i in range(it[2], it[2] + it[3])) for it in items], np.int64) \
        if items else np.zeros(0, np.int64)
    order = np.argsort(-cost, kind="stable")
    items_np = np.array(items, np.int32).reshape(-1, 4)[order] if items else np.zeros((0, 4), np.int32)
    segs_np = np.array([[a, c | (f << 24), mb] for a, c, f, mb in segs], np.uint32).reshape(-1, 3)
    masks_np = np.array(masks, np.uint64) if masks else None
    return PrefillPlan(np.ascontiguousarray(items_np), np.ascontiguousarray(segs_np), masks_np, visited, total)


def plan_from_segments(head_segments, n_heads: int, n: int, s: int) -> PrefillPlan:
    """Native plan: head_segments(h, qt) -> tile segments of the 64-row query
    tile qt (64-key tiles)."""
    n_qt = query_tile_count(n, 64)
    items, segs = [], []
    visited = np.zeros(n_heads, np.int64)
    total = np.zeros(n_heads, np.int64)
    for h in range(n_heads):
        for qt in range(n_qt):
            sg = head_segments(h, qt)
            visited[h] += sum(b - a for a, b in sg)
            total[h] += diagonal_tile(qt, 64, 64, n, s) + 1
        for i in range(0, n_qt, ITEM_ROWS // 64):
            quarters = [head_segments(h, i + k) if i + k < n_qt else None for k in range(ITEM_ROWS // 64)]
            its = _item_segments(quarters, 64 * i, n, s)
            items.append((h, 64 * i, len(segs), len(its)))
            segs.extend((a, c, f, 0) for a, c, f in its)
    return _finish_plan(items, segs, None, visited, total)


def plan_generic(schedules, n_heads: int, n: int, s: int, tq: int, tk: int) -> PrefillPlan:
    """Arbitrary tile sizes: explicit per-row 64-bit column masks per block."""
    if n * s > (1 << 26):
        raise ValueError(f"tile sizes ({tq}, {tk}) need the explicit-mask plan, which is limited to N*S <= 2^26")
    n_qt = query_tile_count(n, tq)
    n_kb = -(-s // 64)
    items, segs, masks = [], [], []
    visited = np.zeros(n_heads, np.int64)
    total = np.zeros(n_heads, np.int64)
    cols = np.arange(n_kb * 64)
    for h in range(n_heads):
        allow_tile = np.zeros((n_qt, -(-s // tk)), bool)
        for qt in range(n_qt):
            tiles = schedules[(h, qt)]
            allow_tile[qt, tiles] = True
            visited[h] += len(tiles)
            total[h] += diagonal_tile(qt, tq, tk, n, s) + 1
        for row0 in range(0, n, ITEM_ROWS):
            rows = np.arange(row0, min(row0 + ITEM_ROWS, n))
            pos = rows + (s - n)
            tile_of_col = np.minimum(cols // tk, allow_tile.shape[1] - 1)
            ok = allow_tile[rows // tq][:, tile_of_col] & (cols[None, :] < s) & (cols[None, :] <= pos[:, None])
            blk_any = ok.reshape(len(rows), n_kb, 64).any(axis=(0, 2))
            nseg = 0
            first_seg = len(segs)
            for b in np.nonzero(blk_any)[0]:
                bits = ok[:, b * 64:(b + 1) * 64]
                words = (bits.astype(np.uint64) << np.arange(64, dtype=np.uint64)[None, :]).sum(axis=1, dtype=np.uint64)
                block_masks = np.zeros(ITEM_ROWS, np.uint64)
                block_masks[:len(rows)] = words
                segs.append((int(b), 1, 0xF | F_MASKS, len(masks) // ITEM_ROWS))
                masks.extend(block_masks.tolist())
                nseg += 1
            items.append((h, row0, first_seg, nseg))
    return _finish_plan(items, segs, masks, visited, total)


def validate_schedules(schedules: Mapping, n_heads: int, n: int, s: int, tq: int, tk: int) -> dict:
    """attn.py:237-308 checks (same messages), plus the finalize check of
    attn.py:184-188 done up front: every row must see at least one column."""
    n_tiles, n_qt = kv_tile_count(s, tk), query_tile_count(n, tq)
    out = {}
    for h in range(n_heads):
        for qt in range(n_qt):
            tiles = [int(t) for t in schedules[(h, qt)]]
            for a, b in zip(tiles, tiles[1:]):
                if b <= a:
                    raise ValueError(f"schedule must be strictly ascending, got {tiles}")
            diag = diagonal_tile(qt, tq, tk, n, s)
            if any(t < 0 or t >= n_tiles for t in tiles):
                raise ValueError(f"schedule for head {h}, query tile {qt} references a tile outside [0, {n_tiles})")
            if tiles and tiles[-1] > diag:
                raise ValueError(f"schedule for head {h}, query tile {qt} references tile {tiles[-1]} "
                                 f"beyond the causal diagonal {diag}")
            if diag not in tiles:
                raise ValueError(f"schedule for head {h}, query tile {qt} omits the most recent KV tile {diag}")
            if tiles[0] * tk > qt * tq + (s - n):
                raise ValueError("row with no attended positions (denominator is 0)")
            out[(h, qt)] = tiles
    return out


def check_finite_device(w: Workload, q, k, v) -> None:
    """Workload's finiteness rule (attn.py:54-56) for host torch tensors,
    evaluated on their device copies."""
    if _device.is_torch(w.q) and not w.q.is_cuda:
        for name, t in (("q", q), ("k", k), ("v", v)):
            if not bool(_device.all_finite(t)):
                raise ValueError(f"non-finite values in {name}")


def run_prefill(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, plan: PrefillPlan, scale: float) -> torch.Tensor:
    """Launch K4 on device tensors q [N,H,Dp], k/v [S,Hkv,Dp] (Dp in {64,128})."""
    lib = _lib.load()
    n, h, dp = q.shape
    s, h_kv, _ = k.shape
    out = torch.empty_like(q)
    items, segs, masks = plan.device_arrays(q.device)
    rc = lib.sk_prefill_attn(_device.sk_dtype(q.dtype), q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                             n, s, h, h_kv, dp, C.c_float(scale), items.data_ptr(), plan.n_items, segs.data_ptr(),
                             masks.data_ptr() if masks is not None else None, _device.stream_ptr(q.device))
    _lib.check(rc)
    return out


def run_prefill_paged(pool, hist: int, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, plan: PrefillPlan,
                      scale: float) -> torch.Tensor:
    """K4 over a page pool (chunked prefill): keys [0, hist) from the pool's KV4
    pages, [hist, hist + n) from the chunk's k/v [n, Hkv, Dp]; q [n, H, Dp]."""
    lib = _lib.load()
    n, h, dp = q.shape
    out = torch.empty_like(q)
    items, segs, masks = plan.device_arrays(q.device)
    abi = pool.abi()
    rc = lib.sk_prefill_attn_paged(C.byref(abi), k.shape[1], hist, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                   out.data_ptr(), n, h, C.c_float(scale), items.data_ptr(), plan.n_items,
                                   segs.data_ptr(), masks.data_ptr() if masks is not None else None,
                                   _device.stream_ptr(q.device))
    _lib.check(rc)
    return out


def blockwise_attention(w: Workload, schedules: Mapping[tuple, Sequence[int]], tile_q: int, tile_k: int,
                        stage: str = "attention", *, dtype: torch.dtype | None = None, device=None):
    """attn.py:245-324 on the B200: causal attention over the scheduled KV
    tiles of every (head, query tile).  Returns (output, CostLedger)."""
    if tile_q < 1 or tile_k < 1:
        raise ValueError("tile sizes must be >= 1")
    n, s = w.num_queries, w.num_history
    if s < n:
        raise ValueError(f"history must cover queries, got S={s}, N={n}")
    tiles = validate_schedules(schedules, w.num_heads, n, s, tile_q, tile_k)
    dev = _device.device_of(device if device is not None else (w.q.device if _device.is_torch(w.q) and w.q.is_cuda else None))
    dt = dtype or (w.q.dtype if _device.is_torch(w.q) and w.q.dtype in (torch.float16, torch.bfloat16)
                   else _device.DEFAULT_DTYPE)
    dp = _device.padded_dim(w.head_dim)
    if tile_q == 64 and tile_k == 64:
        plan = plan_from_segments(lambda h, qt: _segments_of(tiles[(h, qt)]), w.num_heads, n, s)
    else:
        plan = plan_generic(tiles, w.num_heads, n, s, tile_q, tile_k)
    q = _device.to_device(w.q, dt, dev, dp)
    k = _device.to_device(w.k, dt, dev, dp)
    v = _device.to_device(w.v, dt, dev, dp)
    check_finite_device(w, q, k, v)
    out = run_prefill(q, k, v, plan, 1.0 / math.sqrt(w.head_dim))[..., :w.head_dim]
    ledger = CostLedger()
    for h in range(w.num_heads):
        for qt in range(query_tile_count(n, tile_q)):
            ledger.record_tiles(stage, h, len(tiles[(h, qt)]), diagonal_tile(qt, tile_q, tile_k, n, s) + 1)
    np_dt = None if _device.is_torch(w.q) else np.asarray(w.q).dtype
    return _device.to_output(out, w.q, np_dt), ledger
