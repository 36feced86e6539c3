"""CPU oracle for the LServe sparse-attention hot path.

TEST INFRASTRUCTURE ONLY.  This module is the checker: it may be imported by
``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` -- nothing in
``paper_2502_14866_b200`` imports it, and the product path never falls back
to it.

It restates, in plain numpy, the reference package ``sparsekv``
(``/root/reference/pkg/src/sparsekv``; cited below as ``attn.py:L`` etc.)
for exactly the functions on the hot path: tile geometry and blockwise
online-softmax attention, static Lambda-shaped streaming schedules, the
two-way paged / quantised KV store with per-logical-page key bounds, the
Eq. 2 page selector with top-K, pins and reuse, and the prefill/decode
engine with its tile ledger.  The code is a restatement (own structure,
same arithmetic), not a copy.

Parity is pinned: ``tests/golden/make_golden.py`` imports the real
reference in the build container and records its outputs on seeded inputs
as ``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this
oracle against them (bit-exact for integers, page statistics, codes and
selections; 1e-12 relative for float outputs).

Working precision follows the reference: arithmetic on the attention path
happens in the dtype of the inputs (``attn.py:262`` / ``engine.py:226``);
the cache and selector work in float64 (``cache.py:33``, ``selector.py:49``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

RETRIEVAL = "retrieval"
STREAMING = "streaming"
PREFILL = "prefill"
DECODE = "decode"

# ---------------------------------------------------------------------------
# tile geometry  (attn.py:90-122)
# ---------------------------------------------------------------------------


def kv_group(head: int, group: int) -> int:
    """attn.py:90-96 -- query head -> KV head, floor(h / n)."""
    return head // group


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def diagonal(qt: int, tq: int, tk: int, n: int, s: int) -> int:
    """attn.py:111-115 -- last KV tile visible to any row of query tile qt."""
    last_row = min((qt + 1) * tq, n) - 1
    return (s - n + last_row) // tk


def dense_tiles(qt: int, tq: int, tk: int, n: int, s: int) -> list[int]:
    """attn.py:118-122 -- a retrieval head visits range(diag + 1)."""
    return list(range(diagonal(qt, tq, tk, n, s) + 1))


# ---------------------------------------------------------------------------
# static sparsity  (heads.py:68-125)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Role:
    """heads.py:22-34 -- one query head's role and Lambda window."""

    head: int
    gate: float
    role: str
    sink: int = 1
    local: int = 2


def assign_roles(gates, sparsity: float, sink: int = 1, local: int = 2) -> list[Role]:
    """heads.py:68-98 -- ceil((1-s)H - 1e-12) heads with the largest gates
    (ties toward the lower index) retrieve; the rest stream."""
    g = [float(x) for x in gates]
    n_ret = math.ceil((1.0 - sparsity) * len(g) - 1e-12)
    ranked = sorted(range(len(g)), key=lambda h: (-g[h], h))[:n_ret]
    keep = set(ranked)
    return [Role(h, g[h], RETRIEVAL if h in keep else STREAMING, sink, local)
            for h in range(len(g))]


def lambda_tiles(seq_tiles: int, sink: int, local: int, qt: int) -> list[int]:
    """heads.py:107-125 -- sink + local window of a streaming head.

    One contiguous run when the two windows touch, else sink then local."""
    d = min(qt, seq_tiles - 1)
    sink_end = min(sink, d + 1)
    local_start = max(d + 1 - local, 0)
    if local_start <= sink_end:
        return list(range(d + 1))
    return list(range(sink_end)) + list(range(local_start, d + 1))


def lambda_segments(seq_tiles: int, sink: int, local: int, qt: int):
    """Segment form of :func:`lambda_tiles` (heads.py:37-65 BlockIterator)."""
    d = min(qt, seq_tiles - 1)
    sink_end = min(sink, d + 1)
    local_start = max(d + 1 - local, 0)
    if local_start <= sink_end:
        return ((0, d + 1),)
    return ((0, sink_end), (local_start, d + 1))


# ---------------------------------------------------------------------------
# tile ledger  (ledger.py:15-83)
# ---------------------------------------------------------------------------


@dataclass
class Tally:
    """ledger.py:15-36 -- visited/total tiles per (stage, head) and
    selector invocations per KV head."""

    tiles: dict = field(default_factory=dict)
    selector: dict = field(default_factory=dict)

    def add(self, stage: str, head: int, visited: int, total: int) -> None:
        if visited < 0 or total < 0 or visited > total:
            raise ValueError(f"invalid tile counts: visited={visited}, total={total}")
        cell = self.tiles.setdefault((stage, head), [0, 0])
        cell[0] += visited
        cell[1] += total

    def add_selector(self, kv: int, count: int = 1) -> None:
        self.selector[kv] = self.selector.get(kv, 0) + count

    def visited(self, stage=None) -> int:
        return sum(v for (st, _), (v, _) in self.tiles.items() if stage in (None, st))

    def total(self, stage=None) -> int:
        return sum(t for (st, _), (_, t) in self.tiles.items() if stage in (None, st))

    def speedup(self, stage=None) -> float:
        v = self.visited(stage)
        return math.nan if v == 0 else self.total(stage) / v


# ---------------------------------------------------------------------------
# attention  (attn.py:128-324)
# ---------------------------------------------------------------------------


def exact_attention(q, k, v, causal: bool = True) -> np.ndarray:
    """attn.py:128-162 -- dense fp64 softmax(q K^T / sqrt(D)) V, GQA, with
    row i seeing history columns <= S - N + i."""
    q = np.asarray(q, np.float64)
    k = np.asarray(k, np.float64)
    v = np.asarray(v, np.float64)
    n, h_q, d = q.shape
    s, h_kv, _ = k.shape
    grp = h_q // h_kv
    out = np.empty((n, h_q, d))
    hidden = (np.arange(s)[None, :] > (np.arange(n)[:, None] + s - n)) if causal else None
    for h in range(h_q):
        sc = (q[:, h] @ k[:, h // grp].T) * (1.0 / math.sqrt(d))
        if hidden is not None:
            sc = np.where(hidden, -np.inf, sc)
        sc = np.exp(sc - sc.max(axis=1, keepdims=True))
        out[:, h] = (sc / sc.sum(axis=1, keepdims=True)) @ v[:, h // grp]
    return out


def online_merge(m, l, o, scores, values):
    """attn.py:191-229 -- fold one block into the running (max, denom, out).

    Rows that have seen nothing keep max=-inf and shift through 0; the
    previous state is rescaled by exp(m_old - m_new) (0 if m_old=-inf)."""
    dt = m.dtype
    m_new = np.maximum(m, scores.max(axis=1))
    shift = np.where(m_new > -np.inf, m_new, 0.0).astype(dt)
    p = np.exp(scores - shift[:, None])
    a = np.where(m > -np.inf, np.exp(m - shift), 0.0).astype(dt)
    return m_new, a * l + p.sum(axis=1), a[:, None] * o + p @ values


def tiled_attention(q, k, v, schedules, tq: int, tk: int, stage: str = "attention"):
    """attn.py:245-324 -- causal attention over the scheduled KV tiles of
    every (head, query tile), merged in ascending tile order in the input
    dtype; the element-wise causal mask is applied only to tiles whose last
    column passes the tile's first query position (attn.py:315).

    Returns (out [N, H, D], Tally)."""
    n, h_q, d = q.shape
    s, h_kv, _ = k.shape
    grp = h_q // h_kv
    dt = q.dtype
    scale = dt.type(1.0 / math.sqrt(d))
    n_kt, n_qt = ceil_div(s, tk), ceil_div(n, tq)
    out = np.zeros((n, h_q, d), dtype=dt)
    tally = Tally()
    for h in range(h_q):
        kh, vh = k[:, h // grp], v[:, h // grp]
        for qt in range(n_qt):
            r0, r1 = qt * tq, min(n, qt * tq + tq)
            pos = np.arange(r0, r1) + (s - n)
            dg = diagonal(qt, tq, tk, n, s)
            tiles = [int(t) for t in schedules[(h, qt)]]
            if any(b <= a for a, b in zip(tiles, tiles[1:])):
                raise ValueError(f"schedule must be strictly ascending, got {tiles}")
            if any(t < 0 or t >= n_kt for t in tiles):
                raise ValueError(f"schedule for head {h}, query tile {qt} references a tile outside [0, {n_kt})")
            if tiles and tiles[-1] > dg:
                raise ValueError(f"schedule for head {h}, query tile {qt} references tile {tiles[-1]} beyond the causal diagonal {dg}")
            if dg not in tiles:
                raise ValueError(f"schedule for head {h}, query tile {qt} omits the most recent KV tile {dg}")
            m = np.full(r1 - r0, -np.inf, dtype=dt)
            l = np.zeros(r1 - r0, dtype=dt)
            o = np.zeros((r1 - r0, d), dtype=dt)
            qr = q[r0:r1, h]
            for t in tiles:
                c0, c1 = t * tk, min(s, t * tk + tk)
                sc = (qr @ kh[c0:c1].T) * scale
                if c1 - 1 > pos[0]:
                    sc = np.where(np.arange(c0, c1)[None, :] > pos[:, None], -np.inf, sc)
                m, l, o = online_merge(m, l, o, sc, vh[c0:c1])
            if np.any(l <= 0):
                raise ValueError("row with no attended positions (denominator is 0)")
            out[r0:r1, h] = o / l[:, None]
            tally.add(stage, h, len(tiles), dg + 1)
    return out, tally


# ---------------------------------------------------------------------------
# paged, quantised KV store  (cache.py:20-329)
# ---------------------------------------------------------------------------


def quantize(raw, bits):
    """cache.py:20-51 -- per-channel asymmetric uniform quantisation.

    scale = (max-min)/(2^b-1) (1 where that is not > 0), zero = min,
    codes = clip(round_half_even((x - zero)/scale), 0, 2^b-1) as uint8.
    bits=None keeps the raw values with scale 1, zero 0."""
    x = np.asarray(raw, np.float64)
    if x.ndim != 2:
        raise ValueError("expected a [tokens, dim] page")
    if not np.isfinite(x).all():
        raise ValueError("non-finite values in page")
    if bits is None:
        return x.copy(), np.ones(x.shape[1]), np.zeros(x.shape[1])
    if not 2 <= bits <= 8:
        raise ValueError(f"bits must be in [2, 8], got {bits}")
    top = (1 << bits) - 1
    lo, hi = x.min(axis=0), x.max(axis=0)
    sc = (hi - lo) / top
    sc = np.where(sc > 0, sc, 1.0)
    return np.clip(np.round((x - lo) / sc), 0, top).astype(np.uint8), sc, lo


def dequantize(codes, scale, zero):
    """cache.py:54-56 -- code * scale + zero in float64."""
    return codes.astype(np.float64) * scale + zero


@dataclass
class Page:
    """cache.py:76-102 -- one physical page: codes, scale/zero for K and V,
    and (dense pool) per-logical-page (k_min, k_max, covered) bounds."""

    index: int
    tokens: int
    k_codes: np.ndarray
    v_codes: np.ndarray
    k_scale: np.ndarray
    k_zero: np.ndarray
    v_scale: np.ndarray
    v_zero: np.ndarray
    bounds: list = field(default_factory=list)  # [(k_min, k_max, covered)]

    def kv(self):
        """cache.py:97-102 -- dequantised (keys, values) of the live slots."""
        t = self.tokens
        return (dequantize(self.k_codes[:t], self.k_scale, self.k_zero),
                dequantize(self.v_codes[:t], self.v_scale, self.v_zero))


class PagedHead:
    """cache.py:143-274 -- the pages of one KV head in one pool.

    The open tail page keeps raw staging; every append re-quantises the
    whole open page and recomputes its logical bounds (cache.py:211-251).
    A streaming head keeps only index < sink or index >= count - local
    after each append (cache.py:253-261)."""

    def __init__(self, page: int, logical: int, bits, with_bounds: bool, window=None):
        if page % logical:
            raise ValueError("logical page size must divide physical page size")
        self.page, self.logical, self.bits = page, logical, bits
        self.with_bounds, self.window = with_bounds, window
        self.num_tokens = 0
        self.pages: dict[int, Page] = {}
        self._raw_k = None
        self._raw_v = None

    @property
    def page_count(self) -> int:
        return ceil_div(self.num_tokens, self.page) if self.num_tokens else 0

    def live(self) -> list[Page]:
        return [self.pages[i] for i in sorted(self.pages)]

    def append(self, keys, values) -> None:
        keys = np.asarray(keys, np.float64)
        values = np.asarray(values, np.float64)
        if keys.ndim != 2 or keys.shape != values.shape:
            raise ValueError("keys/values must both be [m, dim]")
        if keys.shape[0] < 1:
            raise ValueError("append requires at least one token")
        if not (np.isfinite(keys).all() and np.isfinite(values).all()):
            raise ValueError("non-finite keys or values")
        if self._raw_k is None and self.num_tokens % self.page:
            raise ValueError("cannot append into a partial page restored from a snapshot: its raw staging is gone")
        done = 0
        while done < len(keys):
            if self._raw_k is None:
                self._raw_k = np.empty((0, keys.shape[1]))
                self._raw_v = np.empty((0, keys.shape[1]))
            take = min(self.page - len(self._raw_k), len(keys) - done)
            self._raw_k = np.concatenate([self._raw_k, keys[done:done + take]])
            self._raw_v = np.concatenate([self._raw_v, values[done:done + take]])
            done += take
            self.num_tokens += take
            self._seal_open_page()
            if len(self._raw_k) == self.page:
                self._raw_k = self._raw_v = None
        if self.window is not None:
            sink, local = self.window
            cnt = self.page_count
            for i in [i for i in self.pages if sink <= i < cnt - local]:
                del self.pages[i]

    def _seal_open_page(self) -> None:
        idx = (self.num_tokens - 1) // self.page
        kc, ks, kz = quantize(self._raw_k, self.bits)
        vc, vs, vz = quantize(self._raw_v, self.bits)
        bounds = []
        if self.with_bounds:
            for a in range(0, len(self._raw_k), self.logical):
                blk = self._raw_k[a:a + self.logical]
                bounds.append((blk.min(axis=0), blk.max(axis=0), len(blk)))
        self.pages[idx] = Page(idx, len(self._raw_k), kc, vc, ks, kz, vs, vz, bounds)


class Pools:
    """cache.py:277-329 -- dense pool (with bounds) and streaming pool."""

    def __init__(self, page, logical, bits, dense, streaming, sink=1, local=2):
        both = set(dense) & set(streaming)
        if both:
            raise ValueError(f"heads in both pools: {sorted(both)}")
        self.dense = {h: PagedHead(page, logical, bits, True) for h in sorted(set(dense))}
        self.streaming = {h: PagedHead(page, logical, bits, False, (sink, local))
                          for h in sorted(set(streaming))}

    def head(self, kv: int) -> PagedHead:
        if kv in self.dense:
            return self.dense[kv]
        if kv in self.streaming:
            return self.streaming[kv]
        raise KeyError(f"KV head {kv} is in neither pool")

    @property
    def num_tokens(self) -> int:
        counts = {h.num_tokens for h in list(self.dense.values()) + list(self.streaming.values())}
        if not counts:
            return 0
        if len(counts) != 1:
            raise ValueError(f"pools out of sync: token counts {sorted(counts)}")
        return counts.pop()


# ---------------------------------------------------------------------------
# page selector  (selector.py:22-189)
# ---------------------------------------------------------------------------


def eq2_scores(q_rows, pages: list[Page]) -> np.ndarray:
    """selector.py:39-72 -- Eq. 2 per logical page as
    q . centre + |q| . radius (fp64), max over the group rows, then max
    over each physical page's logical pages."""
    q = np.asarray(q_rows, np.float64)
    if q.ndim == 1:
        q = q[None, :]
    lo, hi, owner = [], [], []
    for i, pg in enumerate(pages):
        if not pg.bounds:
            raise ValueError(f"page {pg.index} carries no key statistics")
        for kmin, kmax, _ in pg.bounds:
            lo.append(kmin)
            hi.append(kmax)
            owner.append(i)
    lo, hi = np.asarray(lo), np.asarray(hi)
    logical = (q @ ((hi + lo) * 0.5).T + np.abs(q) @ ((hi - lo) * 0.5).T).max(axis=0)
    best = np.full(len(pages), -np.inf)
    np.maximum.at(best, np.asarray(owner), logical)
    return best


def eq2_scalar(q, kmin, kmax) -> float:
    """selector.py:22-29 -- sum_i max(q_i kmax_i, q_i kmin_i)."""
    q = np.asarray(q, np.float64)
    return float(np.maximum(q * kmax, q * kmin).sum())


def pins(n: int) -> list[int]:
    """selector.py:75-78 -- {0, n-2, n-1} within [0, n), ascending."""
    return sorted({p for p in (0, max(n - 2, 0), n - 1) if 0 <= p < n})


def top_pages(q_rows, pages: list[Page], budget: int, page: int) -> list[int]:
    """selector.py:81-108 -- K = ceil(budget/page); all pages if K >= n;
    pins only if no free slot; else pins + the best (K - |pins|) others by
    (-score, index); returned ascending."""
    if budget < page:
        raise ValueError(f"budget {budget} is below one page ({page} tokens)")
    n = len(pages)
    if n == 0:
        raise ValueError("no pages to select from")
    k = ceil_div(budget, page)
    if k >= n:
        return list(range(n))
    pinned = pins(n)
    free = max(k - len(pinned), 0)
    if free == 0:
        return pinned
    sc = eq2_scores(q_rows, pages)
    others = sorted((i for i in range(n) if i not in pinned), key=lambda i: (-sc[i], i))
    return sorted(set(pinned) | set(others[:free]))


@dataclass
class Reuse:
    """selector.py:111-125 -- cached selection and its reuse window."""

    pages: list
    start: int
    interval: int
    budget: int

    def covers(self, step: int, budget: int, interval: int) -> bool:
        return (self.budget == budget and self.interval == interval
                and self.start <= step < self.start + interval)


def reuse_or_select(state, step, q_rows, pages, budget, interval, page):
    """selector.py:128-157 -- reuse the cached list object inside its
    window, else reselect with the window starting at ``step``."""
    if interval < 1:
        raise ValueError(f"reuse interval must be >= 1, got {interval}")
    if state is not None and state.covers(step, budget, interval):
        return state.pages, state, False
    chosen = top_pages(q_rows, pages, budget, page)
    return chosen, Reuse(chosen, step, interval, budget), True


def exact_top_pages(q_rows, keys, budget: int, page: int) -> list[int]:
    """selector.py:160-189 -- brute force: rank pages by their best exact
    token score; same pins / top-K rule."""
    q = np.asarray(q_rows, np.float64)
    if q.ndim == 1:
        q = q[None, :]
    keys = np.asarray(keys, np.float64)
    n = ceil_div(keys.shape[0], page)
    k = ceil_div(budget, page)
    if k >= n:
        return list(range(n))
    tok = (q @ keys.T).max(axis=0)
    best = [tok[p * page:(p + 1) * page].max() for p in range(n)]
    pinned = pins(n)
    free = max(k - len(pinned), 0)
    others = sorted((i for i in range(n) if i not in pinned), key=lambda i: (-best[i], i))
    return sorted(set(pinned) | set(others[:free]))


# ---------------------------------------------------------------------------
# engine  (engine.py:30-310)
# ---------------------------------------------------------------------------


@dataclass
class Config:
    """engine.py:30-67 -- the knobs the hot path reads."""

    physical_page: int = 64
    logical_page: int = 16
    quant_bits: int | None = 4
    budget_tokens: int = 4096
    reuse_interval: int = 4
    sink_blocks: int = 1
    local_blocks: int = 2
    target_sparsity: float = 0.5
    tile_q_prefill: int = 64

    def __post_init__(self):
        if self.quant_bits == 0:
            self.quant_bits = None


@dataclass
class Step:
    """engine.py:101-105 -- one decode step's outputs."""

    output: np.ndarray
    tables: list  # per query head: tuple of page indices
    invoked: dict


class OracleEngine:
    """engine.py:108-286 -- one layer of one sequence."""

    def __init__(self, cfg: Config, roles: list[Role]):
        self.cfg, self.roles = cfg, roles
        self.pools: Pools | None = None
        self.tally = Tally()
        self.reuse: dict[int, Reuse] = {}
        self.steps = 0
        self.grp = None

    def _dense(self, h_kv: int) -> set[int]:
        """engine.py:126-132 -- a KV head is dense iff any query head of its
        group retrieves."""
        g = self.grp
        return {kv for kv in range(h_kv)
                if any(self.roles[h].role == RETRIEVAL for h in range(kv * g, kv * g + g))}

    def _new_pools(self, h_kv: int) -> None:
        c = self.cfg
        dense = self._dense(h_kv)
        self.pools = Pools(c.physical_page, c.logical_page, c.quant_bits, dense,
                           set(range(h_kv)) - dense, c.sink_blocks, c.local_blocks)

    def schedules(self, n: int, s: int) -> dict:
        """engine.py:152-165 -- dense heads: range(diag+1); streaming heads:
        sink + local around the diagonal."""
        c = self.cfg
        tq, tk = c.tile_q_prefill, c.physical_page
        n_kt = ceil_div(s, tk)
        out = {}
        for r in self.roles:
            for qt in range(ceil_div(n, tq)):
                dg = diagonal(qt, tq, tk, n, s)
                out[(r.head, qt)] = (list(range(dg + 1)) if r.role == RETRIEVAL
                                     else lambda_tiles(n_kt, r.sink, r.local, dg))
        return out

    def prefill(self, q, k, v) -> np.ndarray:
        """engine.py:136-173 -- blockwise attention on raw K/V, then a fresh
        cache filled with the raw history."""
        if len(self.roles) != q.shape[1]:
            raise ValueError(f"{len(self.roles)} profiles for {q.shape[1]} heads")
        self.grp = q.shape[1] // k.shape[1]
        self._new_pools(k.shape[1])
        out, delta = tiled_attention(q, k, v, self.schedules(q.shape[0], k.shape[0]),
                                     self.cfg.tile_q_prefill, self.cfg.physical_page, PREFILL)
        for (st, h), (vis, tot) in delta.tiles.items():
            self.tally.add(st, h, vis, tot)
        for kv in range(k.shape[1]):
            self.pools.head(kv).append(k[:, kv], v[:, kv])
        return out

    def prefill_chunk(self, q, k, v) -> np.ndarray:
        """Continued prefill (an extension: the reference has no such entry
        point; it composes the reference's own pieces).  The chunk's queries
        sit at positions S0..S0+n-1 and attend, under the static schedules of
        an (n, S0+n) workload (engine.py:152-165), a history made of the
        cached pages dequantised and cast to the q dtype exactly as the
        decode path reads them (engine.py:250-262, cache.py:97-102) followed
        by the chunk's raw K/V; the chunk is then appended (cache.py:189-261).
        A schedule that reaches an evicted page raises, like the reference's
        page lookup would."""
        if self.pools is None or self.pools.num_tokens == 0:
            return self.prefill(q, k, v)
        c = self.cfg
        dt = q.dtype
        n, h_kv = q.shape[0], k.shape[1]
        s0 = self.pools.num_tokens
        s = s0 + n
        kf = np.zeros((s, h_kv, q.shape[2]), dtype=dt)
        vf = np.zeros_like(kf)
        resident = {}
        for kv in range(h_kv):
            head = self.pools.head(kv)
            resident[kv] = set(head.pages)
            for i, pg in head.pages.items():
                kk, vv = pg.kv()
                kf[i * c.physical_page:i * c.physical_page + pg.tokens, kv] = kk.astype(dt)
                vf[i * c.physical_page:i * c.physical_page + pg.tokens, kv] = vv.astype(dt)
        kf[s0:] = k.astype(dt)
        vf[s0:] = v.astype(dt)
        sched = self.schedules(n, s)
        g = self.grp
        for (h, qt), tiles in sched.items():
            miss = [t for t in tiles if t * c.physical_page < s0 and t not in resident[h // g]]
            if miss:
                raise ValueError(f"head {h}, query tile {qt} needs evicted pages {miss}")
        out, delta = tiled_attention(q, kf, vf, sched, c.tile_q_prefill, c.physical_page, PREFILL)
        for (st, h), (vis, tot) in delta.tiles.items():
            self.tally.add(st, h, vis, tot)
        for kv in range(h_kv):
            self.pools.head(kv).append(k[:, kv], v[:, kv])
        return out

    def load_context(self, k, v) -> None:
        """engine.py:175-204 -- cache only, no attention."""
        self.grp = len(self.roles) // k.shape[1]
        self._new_pools(k.shape[1])
        for kv in range(k.shape[1]):
            self.pools.head(kv).append(k[:, kv], v[:, kv])

    def decode_step(self, q, k_new, v_new) -> Step:
        """engine.py:208-286 -- select (retrieval rows only, fp64) per dense
        KV head with reuse; attend each head's pages in ascending order over
        dequantised pages cast to the q dtype, then the raw new token; record
        (visited, page_count-before-append); append afterwards."""
        if self.pools is None or self.pools.num_tokens == 0:
            raise ValueError("decode_step requires a non-empty cache")
        c = self.cfg
        h_q, d = q.shape
        h_kv = k_new.shape[0]
        self.grp = g = h_q // h_kv
        dt = q.dtype
        scale = dt.type(1.0 / np.sqrt(d))
        n_pages = ceil_div(self.pools.num_tokens, c.physical_page)
        chosen, invoked = {}, {}
        for kv in sorted(self.pools.dense):
            rows = [h for h in range(kv * g, kv * g + g) if self.roles[h].role == RETRIEVAL]
            if not rows:
                continue
            sel, st, ran = reuse_or_select(self.reuse.get(kv), self.steps,
                                           q[rows].astype(np.float64),
                                           self.pools.dense[kv].live(), c.budget_tokens,
                                           c.reuse_interval, c.physical_page)
            self.reuse[kv], chosen[kv], invoked[kv] = st, sel, ran
            if ran:
                self.tally.add_selector(kv)
        out = np.empty((h_q, d), dtype=dt)
        tables = []
        for h in range(h_q):
            kv = h // g
            r = self.roles[h]
            idx = chosen[kv] if r.role == RETRIEVAL else lambda_tiles(n_pages, r.sink, r.local, n_pages - 1)
            head = self.pools.head(kv)
            m = np.full(1, -np.inf, dtype=dt)
            l = np.zeros(1, dtype=dt)
            o = np.zeros((1, d), dtype=dt)
            qr = q[h][None, :]
            for p in idx:
                kk, vv = head.pages[p].kv()
                m, l, o = online_merge(m, l, o, (qr @ kk.astype(dt).T) * scale, vv.astype(dt))
            m, l, o = online_merge(m, l, o, (qr @ k_new[kv].astype(dt)[:, None]) * scale,
                                   v_new[kv][None, :].astype(dt))
            if np.any(l <= 0):
                raise ValueError("row with no attended positions (denominator is 0)")
            out[h] = (o / l[:, None])[0]
            tables.append(tuple(int(p) for p in idx))
            self.tally.add(DECODE, h, len(idx), n_pages)
        for kv in range(h_kv):
            self.pools.head(kv).append(k_new[kv][None, :], v_new[kv][None, :])
        self.steps += 1
        return Step(out, tables, invoked)
