"""Planted-needle workloads for selection-recall checks.

Two generators:

* :func:`gen_workload` restates the reference generator
  (``sparsekv.workloads``, workloads.py:74-186) on the host: same numpy RNG
  calls in the same order, same needle placement and planting rule, so a
  spec yields the reference's arrays bit for bit (pinned by
  tests/golden/workloads.json).  The box-score scan is vectorised; each
  score is still one numpy reduction over a contiguous D-vector, as in the
  reference, so the planting coefficient is identical.
* :func:`gen_needles_device` builds a batch of independent trials directly
  on the GPU at long contexts (128k+), one trial per pool stream, with the
  same construction.  Its RNG is torch's, so its tensors are not the
  reference's; the needles are planted against the box scores of the keys
  *as stored* (rounded to the pool dtype), so the margin guarantee holds for
  what the device selector sees.
"""

from __future__ import annotations

import json
import math
from dataclasses import asdict, dataclass
from pathlib import Path

import numpy as np
import torch

from . import _device
from .attn import Workload

RANDOM = "random"
NEEDLE = "needle"
CLUSTERED = "clustered_needles"
KINDS = (RANDOM, NEEDLE, CLUSTERED)


@dataclass(frozen=True)
class WorkloadSpec:
    """workloads.py:28-60."""

    kind: str = RANDOM
    num_history: int = 1024
    num_queries: int = 1
    num_heads: int = 1
    num_kv_heads: int = 1
    head_dim: int = 16
    needle_margin: float = 1.0
    cluster_span: int = 1
    physical_page: int = 64
    logical_page: int = 16
    seed: int = 0

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown workload kind {self.kind!r}")
        if min(self.num_history, self.num_queries, self.num_heads, self.num_kv_heads, self.head_dim) < 1:
            raise ValueError("all dimensions must be positive")
        if self.num_heads % self.num_kv_heads != 0:
            raise ValueError("num_heads must be a multiple of num_kv_heads")
        if self.num_history < self.num_queries:
            raise ValueError("history must cover the query tokens")
        if self.physical_page % self.logical_page != 0:
            raise ValueError("logical page must divide physical page")
        if self.cluster_span < 1:
            raise ValueError("cluster_span must be >= 1")

    def to_dict(self) -> dict:
        return asdict(self)

    @classmethod
    def from_json(cls, path) -> "WorkloadSpec":
        return cls(**json.loads(Path(path).read_text()))


@dataclass(frozen=True)
class GroundTruth:
    """workloads.py:63-70."""

    kind: str
    needle_positions: tuple = ()
    needle_pages: tuple = ()


def _free_pages(num_history: int, page: int) -> list:
    """Full pages away from the pins {0, n-2, n-1} (workloads.py:106-115)."""
    n = math.ceil(num_history / page)
    free = [p for p in range(n) if p != 0 and p < n - 2 and (p + 1) * page <= num_history]
    if not free:
        free = [p for p in range(n) if (p + 1) * page <= num_history]
    if not free:
        raise ValueError(f"history of {num_history} tokens has no full page to plant in")
    return free


def _needle_positions(spec: WorkloadSpec, rng: np.random.Generator) -> list:
    """workloads.py:102-136: one needle in a random free page, or one needle
    per logical page across `cluster_span` consecutive free pages."""
    n_p, n_l = spec.physical_page, spec.logical_page
    free = _free_pages(spec.num_history, n_p)
    if spec.kind == NEEDLE:
        page = int(rng.choice(free))
        return [page * n_p + int(rng.integers(n_p))]
    span = spec.cluster_span
    fs = set(free)
    starts = [p for p in free if all(pp in fs for pp in range(p, p + span))]
    if not starts:
        raise ValueError(f"no room for a {span}-page cluster in {math.ceil(spec.num_history / n_p)} pages")
    start = int(rng.choice(starts))
    out = []
    for page in range(start, start + span):
        for logical in range(n_p // n_l):
            out.append(page * n_p + logical * n_l + int(rng.integers(n_l)))
    return out


def max_box_score(keys: np.ndarray, group_q: np.ndarray, page: int, exclude) -> float:
    """workloads.py:167-186 -- max over non-excluded pages of the group-reduced
    bounding-box score.  Full pages are scored in one batched reduction whose
    per-(page, row) sums run over the same contiguous D-vectors as the
    reference's per-page loop."""
    n = keys.shape[0]
    full = n // page
    best = -math.inf
    keep = np.array([p not in exclude for p in range(full)], bool)
    if full and keep.any():
        blk = keys[:full * page].reshape(full, page, keys.shape[1])[keep]
        lo, hi = blk.min(axis=1), blk.max(axis=1)
        sc = np.maximum(group_q[None] * hi[:, None], group_q[None] * lo[:, None]).sum(axis=2)
        best = float(sc.max())
    if n % page and full not in exclude:
        chunk = keys[full * page:]
        sc = np.maximum(group_q * chunk.max(axis=0), group_q * chunk.min(axis=0)).sum(axis=1).max()
        best = max(best, float(sc))
    return best


def _plant(spec: WorkloadSpec, keys: np.ndarray, group_q: np.ndarray, positions: list) -> None:
    """workloads.py:139-164: overwrite the planted keys with coeff * (the
    longest probe row), coeff chosen so the needle beats every needle-free
    box (physical pages for NEEDLE, logical pages for CLUSTERED) by the margin."""
    if spec.needle_margin <= 0:
        raise ValueError(f"needle margin must be positive, got {spec.needle_margin}")
    norms = np.linalg.norm(group_q, axis=1)
    best = int(np.argmax(norms))
    if norms[best] <= 1e-9:
        raise ValueError("needle cannot dominate: probe query is (numerically) zero, "
                         f"head dim {spec.head_dim} gives it no direction to exploit")
    direction = group_q[best]
    page = spec.physical_page if spec.kind == NEEDLE else spec.logical_page
    exclude = {p // page for p in positions}
    target = max_box_score(keys, group_q, page, exclude) + spec.needle_margin
    coeff = target / float(direction @ direction)
    if not math.isfinite(coeff):
        raise ValueError("needle cannot dominate: non-finite scaling required")
    for pos in positions:
        keys[pos] = coeff * direction


def gen_workload(spec: WorkloadSpec):
    """workloads.py:74-99 -> (Workload of float64 numpy arrays, GroundTruth)."""
    rng = np.random.default_rng(spec.seed)
    s, n = spec.num_history, spec.num_queries
    q = rng.standard_normal((n, spec.num_heads, spec.head_dim))
    k = rng.standard_normal((s, spec.num_kv_heads, spec.head_dim))
    v = rng.standard_normal((s, spec.num_kv_heads, spec.head_dim))
    if spec.kind == RANDOM:
        return Workload(q, k, v), GroundTruth(kind=spec.kind)
    positions = _needle_positions(spec, rng)
    probe = q[-1]
    g = spec.num_heads // spec.num_kv_heads
    for kv in range(spec.num_kv_heads):
        kk = np.ascontiguousarray(k[:, kv, :])
        _plant(spec, kk, probe[kv * g:(kv + 1) * g], positions)
        k[:, kv, :] = kk
    pages = tuple(sorted({p // spec.physical_page for p in positions}))
    return Workload(q, k, v), GroundTruth(spec.kind, tuple(positions), pages)


# ---------------------------------------------------------------------------
# device batch generator
# ---------------------------------------------------------------------------


@dataclass
class NeedleBatch:
    """`trials` independent needle workloads, one per stream.

    keys / values: device [S, trials, Dp] (pool dtype, zero padded channels);
    probes: device [trials, group, Dp]; positions: host [trials, n_needles]."""

    keys: torch.Tensor
    values: torch.Tensor
    probes: torch.Tensor
    positions: np.ndarray
    kind: str
    physical_page: int
    logical_page: int


def _box_scores_device(keys: torch.Tensor, probes: torch.Tensor, page: int) -> torch.Tensor:
    """fp64 group-reduced box score of every page-sized block: [trials, n_blocks]
    (keys [S, T, D], the last partial block included)."""
    s, t, d = keys.shape
    nb = -(-s // page)
    pad = nb * page - s
    k64 = keys.double()
    if pad:  # repeat the last key: leaves min/max of the partial block unchanged
        k64 = torch.cat([k64, k64[-1:].expand(pad, t, d)])
    blk = k64.view(nb, page, t, d)
    lo, hi = blk.amin(1), blk.amax(1)  # [nb, T, D]
    q = probes.double()  # [T, G, D]
    sc = torch.maximum(q[None] * hi[:, :, None], q[None] * lo[:, :, None]).sum(-1)  # [nb, T, G]
    return sc.amax(-1).T.contiguous()  # [T, nb]


def gen_needles_device(kind: str, trials: int, num_history: int, head_dim: int, group: int = 1, *,
                       margin: float = 1.0, cluster_span: int = 1, physical_page: int = 64, logical_page: int = 16,
                       seed: int = 0, dtype: torch.dtype = _device.DEFAULT_DTYPE, device=None) -> NeedleBatch:
    """Device-side batch of NEEDLE / CLUSTERED trials (the construction of
    workloads.py:74-186 with torch's RNG), planted against the stored keys."""
    if kind not in (NEEDLE, CLUSTERED):
        raise ValueError(f"device generator plants needles; got kind {kind!r}")
    if margin <= 0:
        raise ValueError(f"needle margin must be positive, got {margin}")
    if physical_page % logical_page:
        raise ValueError("logical page must divide physical page")
    dev = _device.device_of(device)
    dp = _device.padded_dim(head_dim)
    gen = torch.Generator(device=dev).manual_seed(seed)
    rng = np.random.default_rng(seed)
    keys = torch.zeros((num_history, trials, dp), dtype=dtype, device=dev)
    values = torch.zeros_like(keys)
    probes = torch.zeros((trials, group, dp), dtype=dtype, device=dev)
    keys[..., :head_dim] = torch.randn((num_history, trials, head_dim), generator=gen, device=dev).to(dtype)
    values[..., :head_dim] = torch.randn((num_history, trials, head_dim), generator=gen, device=dev).to(dtype)
    probes[..., :head_dim] = torch.randn((trials, group, head_dim), generator=gen, device=dev).to(dtype)
    spec = WorkloadSpec(kind, num_history, 1, 1, 1, head_dim, margin, cluster_span, physical_page, logical_page)
    positions = np.array([_needle_positions(spec, rng) for _ in range(trials)], np.int64)
    page = physical_page if kind == NEEDLE else logical_page
    scores = _box_scores_device(keys, probes, page)  # [T, nb]
    excl = torch.zeros_like(scores, dtype=torch.bool)
    rows = torch.arange(trials, device=dev)[:, None].expand(-1, positions.shape[1])
    pos_d = torch.as_tensor(positions, device=dev)
    excl[rows, pos_d // page] = True
    target = scores.masked_fill(excl, -math.inf).amax(1) + margin  # [T]
    q64 = probes.double()
    best = q64.norm(dim=-1).argmax(1)  # longest probe row per trial
    direction = q64[torch.arange(trials, device=dev), best]  # [T, Dp]
    coeff = target / (direction * direction).sum(-1)
    needle = (coeff[:, None] * direction).to(dtype)  # [T, Dp]
    keys[pos_d, rows] = needle[:, None, :].expand(-1, positions.shape[1], -1)
    return NeedleBatch(keys, values, probes, positions, kind, physical_page, logical_page)
