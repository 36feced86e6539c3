"""Two-way paged KV store on the device.

Same API as the reference ``sparsekv.cache`` (cache.py:20-413), re-designed
for the B200: each attention layer owns ONE device pool (``DevicePool``)
holding every (sequence, KV head) "stream" -- an arena of fixed-size page
slots (codes + per-page bounds, fragment-native layout), an int32 page
table per stream, per-logical-page key stats and a raw staging copy of
each stream's open page.  Dense-pool streams keep every page; streaming-pool
streams recycle a ring of sink + local slots (eviction = slot reuse).
Appends run the K1 kernel (csrc/append.cu); the host never touches page
contents except through the read-only views below (PhysicalPage snapshots
for tests, snapshots and inspection).
"""

from __future__ import annotations

import ctypes as C
import json
import weakref
from dataclasses import dataclass, field
from typing import IO, Iterable

import numpy as np
import torch

from . import _device, _lib, layout

# ---------------------------------------------------------------------------
# host-side records (reference cache.py:54-106)
# ---------------------------------------------------------------------------


def dequantize_codes(codes: np.ndarray, scale: np.ndarray, zero: np.ndarray) -> np.ndarray:
    """cache.py:54-56."""
    return codes.astype(np.float64) * scale + zero


@dataclass
class PageStats:
    """cache.py:59-73 -- channel-wise key bounds of one logical page."""

    k_min: np.ndarray
    k_max: np.ndarray
    covered_tokens: int

    @classmethod
    def from_keys(cls, keys) -> "PageStats":
        keys = np.asarray(keys, dtype=np.float64)
        if keys.shape[0] < 1:
            raise ValueError("logical page must contain at least one key")
        return cls(keys.min(axis=0), keys.max(axis=0), keys.shape[0])


@dataclass
class PhysicalPage:
    """cache.py:76-102 -- a host snapshot of one device page."""

    page_id: int
    kv_head: int
    capacity: int
    token_count: int
    k_codes: np.ndarray
    v_codes: np.ndarray
    k_scale: np.ndarray
    k_zero: np.ndarray
    v_scale: np.ndarray
    v_zero: np.ndarray
    stats: list = field(default_factory=list)

    def dequantize(self):
        tc = self.token_count
        return (dequantize_codes(self.k_codes[:tc], self.k_scale, self.k_zero),
                dequantize_codes(self.v_codes[:tc], self.v_scale, self.v_zero))


def dequantize_page(page: PhysicalPage):
    return page.dequantize()


# PhysicalPage snapshot -> (DevicePool, stream) it was read from, kept OUTSIDE
# the record so page.__dict__ holds exactly the reference's fields (callers
# rebuild pages with PhysicalPage(**page.__dict__), test_selector.py:62).
_ORIGIN: dict = {}


def _set_origin(page: PhysicalPage, pool, stream: int) -> None:
    key = id(page)
    _ORIGIN[key] = (pool, stream)
    weakref.finalize(page, _ORIGIN.pop, key, None)


def page_origin(page):
    """(DevicePool, stream) a snapshot page came from, or None."""
    return _ORIGIN.get(id(page))


# ---------------------------------------------------------------------------
# device pool
# ---------------------------------------------------------------------------

_NP = {torch.float16: np.float16, torch.bfloat16: None}


def _np_view(raw_u8: np.ndarray, dtype: torch.dtype) -> np.ndarray:
    """Reinterpret 16-bit device values as float64 numpy values (exact)."""
    u16 = raw_u8.view(np.uint16)
    if dtype == torch.float16:
        return u16.view(np.float16).astype(np.float64)
    return (u16.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def _np_exact(a: np.ndarray, np_dt) -> np.ndarray:
    """a.astype(np_dt), refusing values the pool dtype cannot hold exactly
    (a snapshot restores bit-exact pages or nothing; see allow_input_rounding)."""
    out = np.asarray(a).astype(np_dt)
    if not _device._ALLOW_ROUNDING and not np.array_equal(out.astype(np.float64), np.asarray(a, np.float64)):
        raise ValueError(f"snapshot values are not exactly representable in {np.dtype(np_dt).name} (the pool dtype)")
    return out


class DevicePool:
    """All streams of one attention layer: arena + page tables + stats + staging.

    Stream s (a KV head of a sequence) has kind SK_KIND_DENSE (keeps every
    page, carries logical-page key stats) or SK_KIND_STREAMING (keeps only
    sink + local pages: a ring of sink+local arena slots).  Page tables are
    fully populated for [0, max_pages) when (re)allocated, so appends and
    decode steps never upload anything; capacity grows by doubling."""

    def __init__(self, kinds, head_dim: int, page: int, logical: int, bits, sink: int, local: int,
                 dtype: torch.dtype = _device.DEFAULT_DTYPE, device=None, capacity_tokens: int = 0):
        if page % logical:
            raise ValueError("logical page size must divide physical page size")
        self.kinds = [int(k) for k in kinds]
        self.n_streams = len(self.kinds)
        self.D = head_dim
        self.Dp = _device.padded_dim(head_dim)
        self.P, self.L = page, logical
        self.bits = 0 if bits is None else int(bits)
        self.sink, self.local = sink, local
        self.dtype = dtype
        self.device = _device.device_of(device)
        self.slot_bytes = layout.slot_bytes(self.Dp, self.P, self.bits)
        self.tokens_host = [0] * self.n_streams
        self.tokens = torch.zeros(self.n_streams, dtype=torch.int32, device=self.device)
        self.max_pages = 0
        self._alloc(max(4, -(-max(capacity_tokens, 1) // page)))

    # -- allocation ---------------------------------------------------------
    def _slot_ranges(self, max_pages: int):
        offs, n = [], 0
        for k in self.kinds:
            offs.append(n)
            n += max_pages if k == _lib.SK_KIND_DENSE else self.sink + self.local
        return offs, n

    def _page_table(self, max_pages: int, offs) -> np.ndarray:
        pt = np.empty((self.n_streams, max_pages), np.int32)
        p = np.arange(max_pages)
        for s, k in enumerate(self.kinds):
            if k == _lib.SK_KIND_DENSE:
                pt[s] = offs[s] + p
            else:
                pt[s] = offs[s] + np.where(p < self.sink, p, self.sink + (p - self.sink) % self.local)
        return pt

    def _alloc(self, max_pages: int) -> None:
        offs, n_slots = self._slot_ranges(max_pages)
        dev = self.device
        arena = torch.zeros(n_slots * self.slot_bytes, dtype=torch.uint8, device=dev)
        lp = self.P // self.L
        stats = torch.zeros((self.n_streams, max_pages * lp, 2, self.Dp), dtype=self.dtype, device=dev)
        if self.max_pages:  # grow: move the old contents
            old_offs, _ = self._slot_ranges(self.max_pages)
            a_new = arena.view(n_slots, self.slot_bytes)
            a_old = self.arena.view(-1, self.slot_bytes)
            for s, k in enumerate(self.kinds):
                n = self.max_pages if k == _lib.SK_KIND_DENSE else self.sink + self.local
                a_new[offs[s]:offs[s] + n] = a_old[old_offs[s]:old_offs[s] + n]
            stats[:, :self.max_pages * lp] = self.stats
            staging = self.staging
        else:
            staging = torch.zeros((self.n_streams, 2, self.P, self.Dp), dtype=self.dtype, device=dev)
        self.arena, self.stats, self.staging = arena, stats, staging
        self.slot_offsets = offs
        self.page_table_host = self._page_table(max_pages, offs)
        self.page_table = _device.h2d(self.page_table_host, dev)
        self.kind_dev = _device.h2d(np.array(self.kinds, np.uint8), dev)
        self.max_pages = max_pages

    def reserve(self, tokens: int) -> None:
        need = -(-tokens // self.P)
        if need > self.max_pages:
            mp = self.max_pages
            while mp < need:
                mp *= 2
            self._alloc(mp)

    def matches(self, kinds, head_dim: int, page: int, logical: int, bits, sink: int, local: int, dtype) -> bool:
        """Same streams and layout (a pool that can be recycled for a fresh cache)."""
        return (list(kinds) == self.kinds and head_dim == self.D and (page, logical) == (self.P, self.L)
                and (0 if bits is None else int(bits)) == self.bits and (sink, local) == (self.sink, self.local)
                and dtype == self.dtype)

    def reset(self) -> None:
        """Empty every stream (device-side; pages past the token counts are
        never read, and the first append rebuilds page 0 from scratch)."""
        self.tokens.zero_()
        self.tokens_host = [0] * self.n_streams

    # -- ABI view -------------------------------------------------------------
    def decode_workspace(self, group_rows: int) -> torch.Tensor:
        """K3's workspace for this pool (tickets + per-CTA partials), zeroed
        once; the pool's decode launches are stream-ordered, so they share it."""
        need = _lib.load().sk_decode_workspace(self.n_streams, group_rows, self.Dp)
        ws = getattr(self, "_dec_ws", None)
        if ws is None or ws.numel() < need or ws.device != self.device:
            ws = torch.zeros(need, dtype=torch.uint8, device=self.device)
            self._dec_ws = ws
        return ws

    def abi(self, first_stream: int = 0) -> _lib.SkPool:
        s = first_stream
        return _lib.SkPool(
            _device.sk_dtype(self.dtype), self.Dp, self.P, self.L, self.bits, self.max_pages, self.sink, self.local,
            self.slot_bytes, self.arena.data_ptr(),
            self.page_table.data_ptr() + 4 * s * self.max_pages,
            self.stats.data_ptr() + self.stats.element_size() * s * self.stats[0].numel(),
            self.staging.data_ptr() + self.staging.element_size() * s * self.staging[0].numel(),
            self.kind_dev.data_ptr() + s)

    # -- append (K1) --------------------------------------------------------------
    def append(self, k: torch.Tensor, v: torch.Tensor, stream_stride: int, token_stride: int, m: int,
               first_stream: int = 0, n_streams: int | None = None) -> None:
        """Append m tokens to streams [first, first+n); k/v are device tensors of
        the pool dtype with element (s, t, c) at s*stream_stride + t*token_stride + c."""
        n = self.n_streams - first_stream if n_streams is None else n_streams
        n0s = {self.tokens_host[s] for s in range(first_stream, first_stream + n)}
        if len(n0s) != 1:
            raise ValueError(f"pools out of sync: token counts {sorted(n0s)}")
        n0 = n0s.pop()
        self.reserve(n0 + m)
        mpt = (n0 % self.P + m + self.P - 1) // self.P
        pool = self.abi(first_stream)
        rc = _lib.load().sk_append_pages(C.byref(pool), n, k.data_ptr(), v.data_ptr(), stream_stride, token_stride,
                                         self.tokens.data_ptr() + 4 * first_stream, m, mpt,
                                         _device.stream_ptr(self.device))
        _lib.check(rc)
        for s in range(first_stream, first_stream + n):
            self.tokens_host[s] += m

    # -- gather (K1b) ------------------------------------------------------------------
    def gather(self, extra_tokens: int = 0):
        """Dequantised history of every stream as device k/v [S0 + extra, Hkv, Dp]
        in the pool dtype (rows >= S0 left for the caller).  Rows of pages a
        streaming stream has evicted are zero: K4 may load them inside a
        key block whose other page is attended (P < 64), and a masked
        column still meets its V row in the P.V product, where recycled
        NaN bits would poison the output.  One K1b launch."""
        counts = set(self.tokens_host)
        if len(counts) != 1:
            raise ValueError(f"pools out of sync: token counts {sorted(counts)}")
        n0 = counts.pop()
        shape = (n0 + extra_tokens, self.n_streams, self.Dp)
        alloc = torch.zeros if any(kd != _lib.SK_KIND_DENSE for kd in self.kinds) else torch.empty
        k = alloc(shape, dtype=self.dtype, device=self.device)
        v = alloc(shape, dtype=self.dtype, device=self.device)
        if n0:
            pool = self.abi()
            rc = _lib.load().sk_gather_pages(C.byref(pool), self.n_streams, n0, k.data_ptr(), v.data_ptr(), self.Dp,
                                             self.n_streams * self.Dp, _device.stream_ptr(self.device))
            _lib.check(rc)
        return k, v

    # -- snapshot restore ---------------------------------------------------------
    def restore_pages(self, s: int, pages: list) -> None:
        """Write reference-shaped PhysicalPages (codes, scale/zero, stats) into
        stream s: the inverse of snapshot_pages.  Values must be exact in the
        pool dtype (they are when the snapshot came from a pool of that
        dtype).  The stream's token count becomes the end of its last page."""
        if not pages:
            return
        n_tok = max(p.page_id * self.P + p.token_count for p in pages)
        self.reserve(n_tok)
        np_dt = np.float16 if self.dtype == torch.float16 else None
        if np_dt is None:
            raise ValueError("snapshot restore supports fp16 pools")
        levels = (1 << self.bits) - 1 if self.bits else 1
        lp = self.P // self.L
        D, Dp = self.D, self.Dp
        slots, raws = [], []
        stats = self.stats[s].view(-1, 2, Dp)
        for pg in pages:
            t = pg.token_count
            pad = lambda a: np.pad(np.asarray(a, np.float64), (0, Dp - D))  # noqa: E731
            if self.bits:
                kc = np.pad(np.asarray(pg.k_codes[:t], np.uint8), ((0, 0), (0, Dp - D)))
                vc = np.pad(np.asarray(pg.v_codes[:t], np.uint8), ((0, 0), (0, Dp - D)))
                bounds = []
                for scale, zero, codes in ((pg.k_scale, pg.k_zero, kc), (pg.v_scale, pg.v_zero, vc)):
                    lo = pad(zero)
                    const = (pad(scale) == 1.0) & (codes.max(axis=0) == 0)  # hi == lo -> scale forced to 1
                    hi = np.where(const, lo, lo + pad(scale) * levels).astype(np_dt)  # nearest: undoes the /levels
                    lo16 = _np_exact(lo, np_dt)
                    # the restored bounds must reproduce the snapshot's scale exactly (cache.py:44-46)
                    sc = (hi.astype(np.float64) - lo16.astype(np.float64)) / levels
                    sc = np.where(sc > 0, sc, 1.0)
                    if not _device._ALLOW_ROUNDING and not np.array_equal(sc[:D], np.asarray(scale, np.float64)):
                        raise ValueError("snapshot scales are not reproducible from bounds in the pool dtype")
                    bounds += [lo16, hi]
                raw = layout.encode_slot(kc, vc, *bounds, Dp, self.P, self.bits, np_dt, self.slot_bytes)
            else:
                kc = _np_exact(np.pad(np.asarray(pg.k_codes[:t], np.float64), ((0, 0), (0, Dp - D))), np_dt)
                vc = _np_exact(np.pad(np.asarray(pg.v_codes[:t], np.float64), ((0, 0), (0, Dp - D))), np_dt)
                raw = layout.encode_slot(kc, vc, None, None, None, None, Dp, self.P, 0, np_dt, self.slot_bytes)
            slots.append(int(self.page_table_host[s, pg.page_id]))
            raws.append(raw)
            for jl, st in enumerate(pg.stats):
                row = _np_exact(np.stack([pad(st.k_min), pad(st.k_max)]), np_dt)
                stats[pg.page_id * lp + jl].copy_(torch.from_numpy(row))
        arena = self.arena.view(-1, self.slot_bytes)
        arena[torch.as_tensor(slots, device=self.device)] = torch.from_numpy(np.stack(raws)).to(self.device)
        self.tokens_host[s] = n_tok
        self.tokens[s] = n_tok

    # -- host views -------------------------------------------------------------
    def page_count(self, s: int) -> int:
        t = self.tokens_host[s]
        return -(-t // self.P) if t else 0

    def live_indices(self, s: int) -> list:
        n = self.page_count(s)
        if self.kinds[s] == _lib.SK_KIND_DENSE:
            return list(range(n))
        return [p for p in range(n) if p < self.sink or p >= n - self.local]

    def snapshot_pages(self, s: int, indices, kv_head: int) -> list:
        """D2H copy + unpack of the given pages of stream s."""
        indices = list(indices)
        if not indices:
            return []
        slots = torch.as_tensor(self.page_table_host[s, indices].astype(np.int64), device=self.device)
        raw = self.arena.view(-1, self.slot_bytes)[slots].cpu().numpy()
        lp = self.P // self.L
        stats_host = None
        if self.kinds[s] == _lib.SK_KIND_DENSE:
            stats_host = self.stats[s].view(-1, 2 * self.Dp).view(torch.int16).cpu().numpy().view(np.uint8)
        levels = (1 << self.bits) - 1 if self.bits else 1
        pages = []
        n_tok = self.tokens_host[s]
        for i, p in enumerate(indices):
            tc = min(self.P, n_tok - p * self.P)
            kc, vc, klo, khi, vlo, vhi = layout.decode_slot(raw[i], self.Dp, self.P, self.bits, np.uint16)
            D = self.D
            if self.bits == 0:
                kcodes = _np_view(np.ascontiguousarray(kc).view(np.uint8), self.dtype).reshape(self.P, self.Dp)[:, :D]
                vcodes = _np_view(np.ascontiguousarray(vc).view(np.uint8), self.dtype).reshape(self.P, self.Dp)[:, :D]
                ks, kz, vs, vz = np.ones(D), np.zeros(D), np.ones(D), np.zeros(D)
            else:
                kcodes, vcodes = kc[:, :D], vc[:, :D]
                f = lambda a: _np_view(np.ascontiguousarray(a).view(np.uint8), self.dtype)[:D]  # noqa: E731
                klo, khi, vlo, vhi = f(klo), f(khi), f(vlo), f(vhi)
                ks = (khi - klo) / levels
                ks = np.where(ks > 0, ks, 1.0)
                vs = (vhi - vlo) / levels
                vs = np.where(vs > 0, vs, 1.0)
                kz, vz = klo, vlo
            st = []
            if stats_host is not None:
                for jl in range(-(-tc // self.L)):
                    row = stats_host[p * lp + jl]
                    vals = _np_view(row, self.dtype).reshape(2, self.Dp)[:, :D]
                    st.append(PageStats(vals[0].copy(), vals[1].copy(), min(self.L, tc - jl * self.L)))
            pg = PhysicalPage(p, kv_head, self.P, tc, np.ascontiguousarray(kcodes[:tc]),
                              np.ascontiguousarray(vcodes[:tc]), ks, kz, vs, vz, st)
            _set_origin(pg, self, s)  # lets select_pages score device-resident pages in place
            pages.append(pg)
        return pages


# ---------------------------------------------------------------------------
# reference-shaped views
# ---------------------------------------------------------------------------


class PageTable:
    """cache.py:109-140 -- token-order live pages with position -> (page_id,
    slot) lookup.

    ``PageTable(page_size)`` is the reference's stand-alone table (register /
    evict / lookup over a dict).  A ``HeadPages`` owns a *view* table instead
    (``PageTable(head)``): its live pages and token count are read from the
    device stream, whose int32 page table (DevicePool.page_table) is what the
    kernels use; register/evict on a view raise, since residency is decided
    by K1's ring eviction (cache.py:253-261)."""

    def __init__(self, page_size_or_head):
        if isinstance(page_size_or_head, HeadPages):
            self._head = page_size_or_head
            self.page_size = self._head.page_size
            self._live = None
        else:
            self._head = None
            self.page_size = int(page_size_or_head)
            self._live: dict = {}  # global page index -> page_id
            self._num_tokens = 0

    @property
    def num_tokens(self) -> int:
        return self._head.num_tokens if self._head is not None else self._num_tokens

    @num_tokens.setter
    def num_tokens(self, n: int) -> None:
        if self._head is not None:
            raise AttributeError("a device-backed page table counts tokens from its stream")
        self._num_tokens = int(n)

    def register(self, page_index: int, page_id: int) -> None:
        if self._head is not None:
            raise TypeError("device-backed page tables are written by K1 appends, not register()")
        self._live[page_index] = page_id

    def evict(self, page_index: int) -> None:
        if self._head is not None:
            raise TypeError("device-backed page tables evict through K1's streaming ring, not evict()")
        del self._live[page_index]

    @property
    def live_indices(self) -> list:
        return self._head._live() if self._head is not None else sorted(self._live)

    @property
    def page_ids(self) -> list:
        # device pages are identified by their global page index (page_id == index)
        if self._head is not None:
            return self._head._live()
        return [self._live[i] for i in sorted(self._live)]

    def lookup(self, position: int):
        if not 0 <= position < self.num_tokens:
            raise IndexError(f"position {position} outside [0, {self.num_tokens})")
        index = position // self.page_size
        if self._head is not None:
            if index not in set(self._head._live()):
                raise KeyError(f"position {position} falls in an evicted page")
            return index, position % self.page_size
        if index not in self._live:
            raise KeyError(f"position {position} falls in an evicted page")
        return self._live[index], position % self.page_size


class HeadPages:
    """cache.py:143-274 -- the pages of one KV head: a view of one device stream.

    Stand-alone construction (as in the reference tests) creates a private
    one-stream DevicePool on first append."""

    def __init__(self, kv_head: int, page_size: int, logical_page: int, bits, with_stats: bool,
                 streaming_window=None, *, pool: DevicePool | None = None, stream: int = 0,
                 dtype: torch.dtype = _device.DEFAULT_DTYPE, device=None):
        if page_size % logical_page != 0:
            raise ValueError("logical page size must divide physical page size")
        self.kv_head, self.page_size, self.logical_page, self.bits = kv_head, page_size, logical_page, bits
        self.with_stats, self.streaming_window = with_stats, streaming_window
        self._pool, self._stream = pool, stream
        self._dtype, self._device = dtype, device
        self.table = PageTable(self)

    @property
    def pool(self) -> DevicePool | None:
        return self._pool

    @property
    def stream(self) -> int:
        return self._stream

    @property
    def num_tokens(self) -> int:
        return self._pool.tokens_host[self._stream] if self._pool else 0

    @property
    def page_count(self) -> int:
        return self._pool.page_count(self._stream) if self._pool else 0

    def _live(self) -> list:
        return self._pool.live_indices(self._stream) if self._pool else []

    def live_pages(self) -> list:
        return self._pool.snapshot_pages(self._stream, self._live(), self.kv_head) if self._pool else []

    def page_at(self, page_index: int) -> PhysicalPage:
        if page_index not in set(self._live()):
            raise KeyError(f"page index {page_index} is not resident")
        return self._pool.snapshot_pages(self._stream, [page_index], self.kv_head)[0]

    def append(self, keys, values) -> None:
        """cache.py:189-223 -- K1 on this stream."""
        if tuple(np.shape(keys)) != tuple(np.shape(values)) or len(np.shape(keys)) != 2:
            raise ValueError("keys/values must both be [m, dim]")
        if np.shape(keys)[0] < 1:
            raise ValueError("append requires at least one token")
        fin = (lambda t: bool(_device.all_finite(t))) if _device.is_torch(keys) else (lambda t: bool(np.isfinite(t).all()))
        if not (fin(keys) and fin(values)):
            raise ValueError("non-finite keys or values")
        if getattr(self, "_restored_partial", False):
            raise ValueError("cannot append into a partial page restored from a snapshot: its raw staging is gone")
        m, d = np.shape(keys)
        if self._pool is None:
            kind = _lib.SK_KIND_STREAMING if self.streaming_window is not None else _lib.SK_KIND_DENSE
            sink, local = self.streaming_window or (1, 1)
            self._pool = DevicePool([kind], d, self.page_size, self.logical_page, self.bits, sink, local,
                                    self._dtype, self._device, capacity_tokens=m)
            self._stream = 0
        pool = self._pool
        if d != pool.D:
            raise ValueError(f"head_dim mismatch: pool holds {pool.D}, got {d}")
        kd = _device.to_device(keys, pool.dtype, pool.device, pool.Dp)
        vd = _device.to_device(values, pool.dtype, pool.device, pool.Dp)
        pool.append(kd, vd, 0, pool.Dp, m, first_stream=self._stream, n_streams=1)

    def gather(self, page_indices: Iterable[int]):
        ks, vs = [], []
        for p in self._pool.snapshot_pages(self._stream, list(page_indices), self.kv_head) if self._pool else []:
            k, v = p.dequantize()
            ks.append(k)
            vs.append(v)
        if not ks:
            return np.empty((0, 0)), np.empty((0, 0))
        return np.concatenate(ks), np.concatenate(vs)


class TwoWayCache:
    """cache.py:277-329 -- dense and streaming pools backed by ONE DevicePool
    (stream index = rank of the KV head among all heads)."""

    def __init__(self, physical_page: int, logical_page: int, quant_bits, dense_heads: Iterable[int],
                 streaming_heads: Iterable[int], sink_blocks: int = 1, local_blocks: int = 2, *,
                 dtype: torch.dtype = _device.DEFAULT_DTYPE, device=None, capacity_tokens: int = 0):
        dense_heads = sorted(set(dense_heads))
        streaming_heads = sorted(set(streaming_heads))
        both = set(dense_heads) & set(streaming_heads)
        if both:
            raise ValueError(f"heads in both pools: {sorted(both)}")
        self.physical_page, self.logical_page, self.quant_bits = physical_page, logical_page, quant_bits
        self.sink_blocks, self.local_blocks = sink_blocks, local_blocks
        self._dtype, self._device, self._capacity = dtype, device, capacity_tokens
        self.heads = sorted(dense_heads + streaming_heads)
        self.stream_of = {kv: i for i, kv in enumerate(self.heads)}
        self._dense = set(dense_heads)
        self.pool: DevicePool | None = None
        self.dense_pool = {kv: HeadPages(kv, physical_page, logical_page, quant_bits, True) for kv in dense_heads}
        self.streaming_pool = {kv: HeadPages(kv, physical_page, logical_page, quant_bits, False,
                                             (sink_blocks, local_blocks)) for kv in streaming_heads}

    def ensure_pool(self, head_dim: int) -> DevicePool:
        if self.pool is None:
            kinds = self.pool_kinds()
            self.pool = DevicePool(kinds, head_dim, self.physical_page, self.logical_page, self.quant_bits,
                                   self.sink_blocks, self.local_blocks, self._dtype, self._device, self._capacity)
            for kv in self.heads:
                hp = self.pool_of(kv)
                hp._pool, hp._stream = self.pool, self.stream_of[kv]
        return self.pool

    def pool_kinds(self) -> list:
        return [_lib.SK_KIND_DENSE if kv in self._dense else _lib.SK_KIND_STREAMING for kv in self.heads]

    def adopt_pool(self, pool: DevicePool) -> DevicePool:
        """Back this cache with an existing (emptied) device pool."""
        if not pool.matches(self.pool_kinds(), pool.D, self.physical_page, self.logical_page, self.quant_bits,
                            self.sink_blocks, self.local_blocks, self._dtype):
            raise ValueError("pool geometry does not match this cache")
        self.pool = pool
        for kv in self.heads:
            hp = self.pool_of(kv)
            hp._pool, hp._stream = pool, self.stream_of[kv]
        return pool

    def pool_of(self, kv_head: int) -> HeadPages:
        if kv_head in self.dense_pool:
            return self.dense_pool[kv_head]
        if kv_head in self.streaming_pool:
            return self.streaming_pool[kv_head]
        raise KeyError(f"KV head {kv_head} is in neither pool")

    def append_tokens(self, kv_head: int, keys, values) -> None:
        hp = self.pool_of(kv_head)
        self.ensure_pool(np.shape(keys)[1])
        hp.append(keys, values)

    def append_all(self, k: torch.Tensor, v: torch.Tensor) -> None:
        """Bulk append of device k/v [m, Hkv, Dp] to every stream (one K1 launch)."""
        pool = self.ensure_pool(self._user_dim or k.shape[2])
        m, h_kv, dp = k.shape
        if h_kv != len(self.heads) or self.heads != list(range(h_kv)):
            raise ValueError("append_all needs KV heads 0..Hkv-1")
        pool.append(k, v, dp, h_kv * dp, m)

    _user_dim = None

    @property
    def num_tokens(self) -> int:
        if self.pool is None:
            return 0
        counts = set(self.pool.tokens_host)
        if len(counts) != 1:
            raise ValueError(f"pools out of sync: token counts {sorted(counts)}")
        return counts.pop()

    # -- snapshot (cache.py:333-413) ---------------------------------------------
    def dump_jsonl(self, fp: IO[str]) -> None:
        header = {"physical_page": self.physical_page, "logical_page": self.logical_page, "bits": self.quant_bits}
        fp.write(json.dumps(header) + "\n")
        for pool_name, pool in (("dense", self.dense_pool), ("streaming", self.streaming_pool)):
            for kv in sorted(pool):
                for page in pool[kv].live_pages():
                    fp.write(json.dumps(_page_record(pool_name, page)) + "\n")


def _load_jsonl(cls, fp: IO[str], *, dtype: torch.dtype = _device.DEFAULT_DTYPE, device=None) -> "TwoWayCache":
    """cache.py:347-368: rebuild a cache from a dump_jsonl snapshot.  Pages go
    back into device pools; a head whose last page is partial refuses further
    appends (its raw staging is gone, cache.py:199-203)."""
    header = json.loads(fp.readline())
    recs = [json.loads(line) for line in fp if line.strip()]
    dense = sorted({r["kv_head"] for r in recs if r["pool"] == "dense"})
    streaming = sorted({r["kv_head"] for r in recs if r["pool"] == "streaming"})
    P = header["physical_page"]
    cap = max([r["page_id"] * P + r["token_count"] for r in recs] or [1])
    cache = cls(P, header["logical_page"], header["bits"], dense, streaming, dtype=dtype, device=device,
                capacity_tokens=cap)
    if not recs:
        return cache
    cache.ensure_pool(len(recs[0]["k_scale"]))
    pool = cache.pool
    for kv in cache.heads:
        mine = [r for r in recs if r["kv_head"] == kv]
        pages = [PhysicalPage(r["page_id"], kv, P, r["token_count"], np.asarray(r["k_codes"]),
                              np.asarray(r["v_codes"]), np.asarray(r["k_scale"]), np.asarray(r["k_zero"]),
                              np.asarray(r["v_scale"]), np.asarray(r["v_zero"]),
                              [PageStats(np.asarray(st["k_min"]), np.asarray(st["k_max"]), st["covered_tokens"])
                               for st in r["stats"]]) for r in mine]
        pool.restore_pages(cache.stream_of[kv], pages)
        hp = cache.pool_of(kv)
        hp._restored_partial = bool(pages) and max(pages, key=lambda p: p.page_id).token_count < P
    return cache


TwoWayCache.load_jsonl = classmethod(_load_jsonl)


def _page_record(pool_name: str, page: PhysicalPage) -> dict:
    as_list = (lambda a: a[:page.token_count].tolist())
    return {
        "pool": pool_name, "kv_head": page.kv_head, "page_id": page.page_id, "token_count": page.token_count,
        "k_codes": as_list(page.k_codes), "v_codes": as_list(page.v_codes),
        "k_scale": page.k_scale.tolist(), "k_zero": page.k_zero.tolist(),
        "v_scale": page.v_scale.tolist(), "v_zero": page.v_zero.tolist(),
        "stats": [{"k_min": s.k_min.tolist(), "k_max": s.k_max.tolist(), "covered_tokens": s.covered_tokens}
                  for s in page.stats],
        "codes_dtype": str(page.k_codes.dtype),
    }


def quantize_page(raw, bits):
    """cache.py:20-51 through K1: one page (<= 128 tokens) is appended to a
    private one-stream pool and read back.  Exact for inputs representable
    in the device dtype (fp16 by default)."""
    raw_np = raw.detach().cpu().numpy() if _device.is_torch(raw) else np.asarray(raw)
    if raw_np.ndim != 2:
        raise ValueError("expected a [tokens, dim] page")
    if not np.isfinite(raw_np).all():
        raise ValueError("non-finite values in page")
    if bits is not None and not 2 <= bits <= 8:
        raise ValueError(f"bits must be in [2, 8], got {bits}")
    t, d = raw_np.shape
    if t > 128:
        raise ValueError("quantize_page on the B200 path takes pages of at most 128 tokens")
    page = 32 if t <= 32 else (64 if t <= 64 else 128)
    head = HeadPages(0, page, page, bits, with_stats=False)
    head.append(raw_np, raw_np)
    pg = head.page_at(0)
    return pg.k_codes, pg.k_scale, pg.k_zero
