"""Selection recall on the B200 selector.

Mirrors the reference's recall machinery -- ``sweeps.clustered_recall``
(sweeps.py:43-97) and the C06 needle check (verify.py:219-248) -- with the
page selection done by K2 over device pools: every trial is one stream of a
raw-page (bits None) pool per paging scheme, K1 fills all of them in one
launch and K2 selects for all of them in one launch per budget.  The
"oracle" entry ranks pages by exact token scores (selector.py:160-189,
``exact_top_k_pages``), computed on the device in fp64 over the keys as
stored.  Keys are stored in the pool dtype, so on reference (float64)
workloads the selections can differ from the reference's where a rounding
flips a near-tie; tests/test_gpu_recall.py bounds that difference.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device, _lib
from .cache import DevicePool
from .selector import pinned_pages, select_streams, selection_size
from .workloads import CLUSTERED, NEEDLE, NeedleBatch, WorkloadSpec, gen_workload

SCHEMES = (("hierarchical", 64, 16), ("flat_coarse", 64, 64), ("flat_fine", 16, 16))


def _pool(keys: torch.Tensor, values: torch.Tensor, page: int, logical: int) -> DevicePool:
    s, t, dp = keys.shape
    pool = DevicePool([_lib.SK_KIND_DENSE] * t, dp, page, logical, None, 1, 1, keys.dtype, keys.device,
                      capacity_tokens=s)
    pool.append(keys, values, dp, t * dp, s)
    return pool


def device_select(pool: DevicePool, probes: torch.Tensor, budget_tokens: int) -> list:
    """K2 over every stream of `pool` with probe rows [T, G, Dp]; returns the
    ascending selected page list of each stream (selector.py:81-108)."""
    t, g, dp = probes.shape
    n_pages = pool.page_count(0)
    k = -(-budget_tokens // pool.P)
    size = selection_size(n_pages, k)
    out = torch.empty((t, max(4, size)), dtype=torch.int32, device=pool.device)
    cnt = torch.empty(t, dtype=torch.int32, device=pool.device)
    mask = torch.full((t,), (1 << g) - 1, dtype=torch.int32, device=pool.device)
    select_streams(pool, probes, g * dp, dp, g, mask, k, out, cnt, max_pages_hint=n_pages)
    out, cnt = out.cpu().numpy(), cnt.cpu().numpy()
    return [out[i, :cnt[i]].tolist() for i in range(t)]


def exact_top_pages(keys: torch.Tensor, probes: torch.Tensor, budget_tokens: int, page: int) -> list:
    """selector.py:160-189 on the device: pages ranked by their best exact
    token score (max over the group), pins + top K-|pins|, ascending."""
    s, t, dp = keys.shape
    n_pages = -(-s // page)
    k = -(-budget_tokens // page)
    if k >= n_pages:
        return [list(range(n_pages))] * t
    tok = torch.einsum("stc,tgc->tgs", keys.double(), probes.double()).amax(1)  # [T, S]
    pad = n_pages * page - s
    if pad:
        tok = torch.cat([tok, tok[:, -1:].expand(-1, pad)], 1)
    ps = tok.view(t, n_pages, page).amax(-1)
    pins = pinned_pages(n_pages)
    free = max(k - len(pins), 0)
    ps[:, pins] = -torch.inf
    order = torch.sort(-ps, dim=1, stable=True).indices[:, :free].cpu().numpy()  # ties -> lower index
    return [sorted(set(pins) | set(order[i].tolist())) for i in range(t)]


def batch_recall(batch: NeedleBatch, budgets, schemes=SCHEMES, oracle_page: int = 64) -> dict:
    """Token-level recall per budget and scheme over every trial of `batch`:
    the fraction of planted positions whose page is selected."""
    pos = batch.positions
    total = pos.size
    pools = {name: (_pool(batch.keys, batch.values, page, logical), page) for name, page, logical in schemes}
    out = {}
    for b in budgets:
        row = {}
        for name, (pool, page) in pools.items():
            sel = device_select(pool, batch.probes, b)
            row[name] = sum(int(p // page in set(sel[i])) for i in range(len(sel)) for p in pos[i]) / total
        orc = exact_top_pages(batch.keys, batch.probes, b, oracle_page)
        row["oracle"] = sum(int(p // oracle_page in set(orc[i])) for i in range(len(orc)) for p in pos[i]) / total
        out[b] = row
    return out


def _reference_batch(specs, dtype, device) -> NeedleBatch:
    """Stack host reference workloads (one KV head each) as pool streams."""
    ws = [gen_workload(s) for s in specs]
    dp = _device.padded_dim(specs[0].head_dim)
    d = specs[0].head_dim
    keys = np.zeros((specs[0].num_history, len(ws), dp))
    vals = np.zeros_like(keys)
    probes = np.zeros((len(ws), specs[0].num_heads, dp))
    for i, (w, _) in enumerate(ws):
        keys[:, i, :d] = w.k[:, 0, :]
        vals[:, i, :d] = w.v[:, 0, :]
        probes[i, :, :d] = w.q[-1]
    dev = _device.device_of(device)
    cast = lambda a: torch.from_numpy(a).to(device=dev, dtype=dtype)  # noqa: E731
    positions = np.array([t.needle_positions for _, t in ws], np.int64)
    return NeedleBatch(cast(keys), cast(vals), cast(probes), positions, specs[0].kind, specs[0].physical_page,
                       specs[0].logical_page)


def clustered_recall(budgets, trials: int, seed: int, num_history: int = 2048, dim: int = 16, cluster_span: int = 2,
                     margin: float = 0.75, schemes=SCHEMES, *, dtype=_device.DEFAULT_DTYPE, device=None) -> dict:
    """sweeps.py:43-97 with K2 doing the selection: the reference's own
    workloads (seeds seed*trials + i), {budget: {scheme: recall, "oracle": r}}."""
    specs = [WorkloadSpec(kind=CLUSTERED, num_history=num_history, num_queries=1, num_heads=1, num_kv_heads=1,
                          head_dim=dim, needle_margin=margin, cluster_span=cluster_span, physical_page=64,
                          logical_page=16, seed=seed * trials + i) for i in range(trials)]
    return batch_recall(_reference_batch(specs, dtype, device), budgets, schemes)


def needle_recall(trials: int, seed: int, num_history: int = 512, dim: int = 16, margin: float = 0.5,
                  budget: int = 256, *, dtype=_device.DEFAULT_DTYPE, device=None) -> dict:
    """verify.py:219-248 (C06) with K2 doing the selection: recall of the
    needle page, the exact-score oracle's recall, and their agreement."""
    specs = [WorkloadSpec(kind=NEEDLE, num_history=num_history, num_queries=1, num_heads=1, num_kv_heads=1,
                          head_dim=dim, needle_margin=margin, physical_page=64, logical_page=16,
                          seed=seed * trials + i) for i in range(trials)]
    batch = _reference_batch(specs, dtype, device)
    pool = _pool(batch.keys, batch.values, 64, 16)
    sel = device_select(pool, batch.probes, budget)
    orc = exact_top_pages(batch.keys, batch.probes, budget, 64)
    pages = batch.positions[:, 0] // 64
    hit = np.array([pages[i] in sel[i] for i in range(trials)])
    ohit = np.array([pages[i] in orc[i] for i in range(trials)])
    return {"trials": trials, "recall": float(hit.mean()), "oracle_recall": float(ohit.mean()),
            "oracle_agreement": float((hit == ohit).mean())}
