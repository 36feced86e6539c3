"""Query-aware page selection (LServe Eq. 2) on the device.

API mirrors the reference ``sparsekv.selector`` (selector.py:22-189).  The
scoring and top-K run in the K2 kernel (csrc/select.cu): tensor-core fp32
scores with a rigorous error bound, the pages near the K-th score rescored
exactly in fp64, the reference's tie-break (lower page index); results are
bit-identical to the reference for inputs exactly representable in the
device dtype.  The two
scalar helpers ``logical_page_score`` / ``physical_page_score`` evaluate
Eq. 2 for a single page on the host, like the reference's.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _device, _lib
from .cache import DevicePool, PageStats, PhysicalPage, page_origin


def logical_page_score(q, stats: PageStats) -> float:
    """selector.py:22-29 -- sum_i max(q_i kmax_i, q_i kmin_i)."""
    q = np.asarray(q, dtype=np.float64)
    if q.shape != stats.k_max.shape:
        raise ValueError(f"query dim {q.shape} does not match stats dim {stats.k_max.shape}")
    return float(np.maximum(q * stats.k_max, q * stats.k_min).sum())


def physical_page_score(q, page: PhysicalPage) -> float:
    """selector.py:32-36."""
    if not page.stats:
        raise ValueError(f"page {page.page_id} carries no key statistics")
    return max(logical_page_score(q, s) for s in page.stats)


def pinned_pages(num_pages: int) -> list:
    """selector.py:75-78 -- sink page + the two most recent pages."""
    return sorted({p for p in (0, max(num_pages - 2, 0), num_pages - 1) if 0 <= p < num_pages})


def selection_size(num_pages: int, budget_pages: int) -> int:
    """Length of select_pages' output (selector.py:97-108)."""
    if budget_pages >= num_pages:
        return num_pages
    return max(budget_pages, len(pinned_pages(num_pages)))


class _Workspace:
    """Per-(device, stream count) select workspace, grown geometrically.  Its
    tickets sit at a fixed offset (sk_select_workspace) and start at zero;
    the kernel re-arms them, so a larger page count only ever reallocates
    when it outgrows the buffer."""

    _by_dev: dict = {}

    @classmethod
    def get(cls, device, n_streams: int, max_pages: int) -> torch.Tensor:
        lib = _lib.load()
        need = lib.sk_select_workspace(n_streams, max_pages)
        key = (str(device), n_streams)
        ws = cls._by_dev.get(key)
        if ws is None or ws.numel() < need:
            pages = max_pages if ws is None else max(max_pages, 2 * cls._pages(ws, n_streams))
            ws = torch.zeros(lib.sk_select_workspace(n_streams, pages), dtype=torch.uint8, device=device)
            cls._by_dev[key] = ws
        return ws

    @staticmethod
    def _pages(ws: torch.Tensor, n_streams: int) -> int:
        return (ws.numel() - _lib.load().sk_select_scores_offset(n_streams)) // (16 * n_streams)


def select_streams(pool: DevicePool, q: torch.Tensor, q_stream_stride: int, q_row_stride: int, group_rows: int,
                   row_mask: torch.Tensor, budget_pages: int, out: torch.Tensor, count: torch.Tensor,
                   first_stream: int = 0, n_streams: int | None = None, invoke: torch.Tensor | None = None,
                   max_pages_hint: int | None = None) -> torch.Tensor:
    """Launch K2 over streams [first, first+n) of `pool`; returns the workspace."""
    n = pool.n_streams - first_stream if n_streams is None else n_streams
    mp = max_pages_hint or max(1, max(pool.page_count(s) for s in range(first_stream, first_stream + n)))
    ws = _Workspace.get(pool.device, n, mp)
    abi = pool.abi(first_stream)
    rc = _lib.load().sk_select_pages(
        C.byref(abi), n, group_rows, q.data_ptr(), q_stream_stride, q_row_stride, row_mask.data_ptr(),
        pool.tokens.data_ptr() + 4 * first_stream, invoke.data_ptr() if invoke is not None else None,
        budget_pages, mp, out.data_ptr(), count.data_ptr(), out.shape[-1], ws.data_ptr(), ws.numel(), 0,
        _device.stream_ptr(pool.device))
    _lib.check(rc)
    return ws


def _pool_for_pages(pages: Sequence[PhysicalPage], page_size: int, device) -> DevicePool:
    """Upload the key stats of an arbitrary page list into a one-stream pool
    (page i -> index i).  Missing logical entries of a short page repeat one
    of its own entries, which leaves the max-reduced page score unchanged."""
    dim = pages[0].stats[0].k_min.shape[0]
    lp = max(len(p.stats) for p in pages)
    logical = max(1, page_size // lp)
    pool = DevicePool([_lib.SK_KIND_DENSE], dim, page_size, logical, None, 1, 1, device=device,
                      capacity_tokens=len(pages) * page_size)
    host = np.zeros((len(pages) * lp, 2, pool.Dp), np.float64)
    for i, p in enumerate(pages):
        for j in range(lp):
            s = p.stats[min(j, len(p.stats) - 1)]
            host[i * lp + j, 0, :dim] = s.k_min
            host[i * lp + j, 1, :dim] = s.k_max
    pool.stats[0, :host.shape[0]] = _device.exact_cast(torch.from_numpy(host).to(pool.device), pool.dtype)
    pool.tokens_host[0] = len(pages) * page_size
    pool.tokens.fill_(len(pages) * page_size)
    return pool


def _select_inputs(q_group, pages: Sequence[PhysicalPage], page_size: int, dev):
    for p in pages:
        if not p.stats:
            raise ValueError(f"page {p.page_id} carries no key statistics")
    q = np.asarray(q_group.detach().cpu() if _device.is_torch(q_group) else q_group, dtype=np.float64)
    if q.ndim == 1:
        q = q[None, :]
    rows = q.shape[0]
    if rows > 32:
        raise ValueError("select_pages on the B200 path takes at most 32 query rows per KV head")
    src = page_origin(pages[0])
    pool = None
    if src is not None and all(page_origin(p) == src for p in pages):
        cand, stream = src
        if [p.page_id for p in pages] == list(range(cand.page_count(stream))) and \
                cand.kinds[stream] == _lib.SK_KIND_DENSE and cand.P == page_size:
            pool, first = cand, stream
    if pool is None:
        pool, first = _pool_for_pages(pages, page_size, dev), 0
    qd = _device.to_device(q, pool.dtype, pool.device, pool.Dp)
    mask = torch.tensor([(1 << rows) - 1], dtype=torch.int64, device=pool.device).to(torch.int32)
    return pool, first, qd, mask, rows


def _run_select(q_group, pages: Sequence[PhysicalPage], budget_pages: int, page_size: int, device=None):
    dev = _device.device_of(device)
    pool, first, qd, mask, rows = _select_inputs(q_group, pages, page_size, dev)
    k_out = max(1, min(budget_pages, len(pages)))
    out = torch.empty((1, max(k_out, 4)), dtype=torch.int32, device=pool.device)
    cnt = torch.empty(1, dtype=torch.int32, device=pool.device)
    ws = select_streams(pool, qd, 0, pool.Dp, rows, mask, budget_pages, out, cnt, first_stream=first,
                        n_streams=1, max_pages_hint=len(pages))
    return out, cnt, ws


def select_pages(q_group, pages: Sequence[PhysicalPage], budget_tokens: int, page_size: int,
                 *, device=None) -> list:
    """selector.py:81-108 -- top-K pages under the token budget, pins included, ascending."""
    if budget_tokens < page_size:
        raise ValueError(f"budget {budget_tokens} is below one page ({page_size} tokens)")
    n = len(pages)
    if n == 0:
        raise ValueError("no pages to select from")
    k = -(-budget_tokens // page_size)
    out, cnt, _ = _run_select(q_group, pages, k, page_size, device)
    c = int(cnt.item())
    return out[0, :c].cpu().tolist()


def score_pages(q_group, pages: Sequence[PhysicalPage], *, device=None) -> np.ndarray:
    """selector.py:39-72 -- fp64 physical-page scores (max over group rows),
    by sk_score_pages (the exact arithmetic K2 ranks its boundary pages with)."""
    pages = list(pages)
    dev = _device.device_of(device)
    pool, first, qd, mask, rows = _select_inputs(q_group, pages, pages[0].capacity, dev)
    out = torch.empty((1, len(pages)), dtype=torch.float64, device=pool.device)
    abi = pool.abi(first)
    rc = _lib.load().sk_score_pages(C.byref(abi), 1, rows, qd.data_ptr(), 0, pool.Dp, mask.data_ptr(),
                                    pool.tokens.data_ptr() + 4 * first, out.data_ptr(), len(pages),
                                    _device.stream_ptr(pool.device))
    _lib.check(rc)
    return out[0].cpu().numpy().copy()


def exact_top_k_pages(q_group, keys, budget_tokens: int, page_size: int, *, device=None) -> list:
    """selector.py:160-189 -- brute-force oracle: pages ranked by their best
    exact token score (fp64 q.k of every stored key, max over the group rows
    and the page), with the selector's pins and tie rule.  Runs on the device
    (fp64 matmul); used to measure selection recall, not on the decode path."""
    if budget_tokens < page_size:
        raise ValueError(f"budget {budget_tokens} is below one page ({page_size} tokens)")
    dev = _device.device_of(device)
    as_t = lambda x: (x.detach() if _device.is_torch(x) else torch.from_numpy(np.asarray(x, np.float64)))  # noqa: E731
    q = as_t(q_group).to(dev, torch.float64)
    if q.ndim == 1:
        q = q[None, :]
    k = as_t(keys).to(dev, torch.float64)
    num_pages = -(-k.shape[0] // page_size)
    kp = -(-budget_tokens // page_size)
    if kp >= num_pages:
        return list(range(num_pages))
    tok = (q @ k.T).amax(0)
    pad = num_pages * page_size - k.shape[0]
    if pad:
        tok = torch.cat([tok, tok.new_full((pad,), -float("inf"))])
    page_scores = tok.view(num_pages, page_size).amax(1).cpu().numpy()
    pins = pinned_pages(num_pages)
    free = max(kp - len(pins), 0)
    cand = [i for i in range(num_pages) if i not in set(pins)]
    cand.sort(key=lambda i: (-page_scores[i], i))
    return sorted(set(pins) | set(cand[:free]))


@dataclass
class SelectionState:
    """selector.py:111-125."""

    selected_pages: list
    chunk_start_step: int
    reuse_interval: int
    budget_tokens: int

    def valid_for(self, step: int, budget_tokens: int, reuse_interval: int) -> bool:
        return (self.budget_tokens == budget_tokens and self.reuse_interval == reuse_interval
                and self.chunk_start_step <= step < self.chunk_start_step + reuse_interval)


def reusable_select(state, step: int, q_group, pages, budget_tokens: int, reuse_interval: int, page_size: int):
    """selector.py:128-157 -- reuse the identical list object within a chunk."""
    if reuse_interval < 1:
        raise ValueError(f"reuse interval must be >= 1, got {reuse_interval}")
    if state is not None and state.valid_for(step, budget_tokens, reuse_interval):
        return state.selected_pages, state, False
    selected = select_pages(q_group, pages, budget_tokens, page_size)
    return selected, SelectionState(selected, step, reuse_interval, budget_tokens), True
