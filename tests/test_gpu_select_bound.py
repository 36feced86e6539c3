"""K2's fp32 tensor-core filter (csrc/select.cu, phase A) against the exact
fp64 page scores (sk_score_pages): the stored error bound must cover the
fp32 score of EVERY page -- the premise that lets the kernel rescore only the
band around the K-th score -- and the selection must equal the oracle's
fp64 ranking (selector.py:39-108) on N(0,1), wide-range (subnormal to
near-overflow) fp16, wide-range bf16 and overflowing bf16 statistics."""

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import sparsekv_oracle as O
from paper_2502_14866_b200 import _device, _lib
from paper_2502_14866_b200.cache import DevicePool
from paper_2502_14866_b200.selector import select_streams

pytestmark = pytest.mark.gpu


def _pool(stats, dtype, page, logical):
    """One dense stream holding the given [n_logical, 2, D] (k_min, k_max) stats."""
    n_log, _, d = stats.shape
    pool = DevicePool([_lib.SK_KIND_DENSE], d, page, logical, None, 1, 1, dtype=dtype, device="cuda:0",
                      capacity_tokens=n_log * logical)
    pool.stats[0, :n_log] = torch.from_numpy(stats).to("cuda:0").to(dtype)
    pool.tokens_host[0] = n_log * logical
    pool.tokens.fill_(n_log * logical)
    return pool


def _run(stats, q, dtype, page, logical, k_pages):
    pool = _pool(stats, dtype, page, logical)
    rows, d = q.shape
    qd = torch.from_numpy(q).to("cuda:0").to(dtype).contiguous()
    mask = torch.tensor([(1 << rows) - 1], dtype=torch.int64, device="cuda:0").to(torch.int32)
    n_pages = stats.shape[0] * logical // page
    out = torch.zeros((1, max(k_pages, 4)), dtype=torch.int32, device="cuda:0")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    ws = select_streams(pool, qd, 0, d, rows, mask, k_pages, out, cnt, n_streams=1, max_pages_hint=n_pages)
    exact = torch.empty((1, n_pages), dtype=torch.float64, device="cuda:0")
    abi = pool.abi()
    _lib.check(_lib.load().sk_score_pages(C.byref(abi), 1, rows, qd.data_ptr(), 0, d, mask.data_ptr(),
                                          pool.tokens.data_ptr(), exact.data_ptr(), n_pages,
                                          _device.stream_ptr(pool.device)))
    off = _lib.load().sk_select_scores_offset(1)
    pairs = ws[off:off + 8 * n_pages].view(torch.float32).view(n_pages, 2).double().cpu().numpy()
    torch.cuda.synchronize()
    sel = out[0, :int(cnt.item())].cpu().tolist()
    return pairs, exact[0].cpu().numpy(), sel


def _oracle_sel(stats_f64, q_f64, page, logical, k_pages):
    lp = page // logical
    pages = [O.Page(i, page, None, None, None, None, None, None,
                    [(stats_f64[i * lp + j, 0], stats_f64[i * lp + j, 1], logical) for j in range(lp)])
             for i in range(stats_f64.shape[0] // lp)]
    return O.top_pages(q_f64, pages, k_pages * page, page)


def _stats_from(a, b):
    lo, hi = np.minimum(a, b), np.maximum(a, b)
    return np.stack([lo, hi], axis=1)


CASES = {
    "normal_f16": torch.float16,
    "wide_f16": torch.float16,
    "wide_bf16": torch.bfloat16,
    "overflow_bf16": torch.bfloat16,
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("d,rows", [(128, 2), (128, 4), (64, 3), (128, 11)])
def test_fp32_filter_bound_covers_exact_scores(case, d, rows):
    dtype = CASES[case]
    rng = np.random.default_rng(hash((case, d, rows)) % 2**32)
    page, logical, n_pages = 64, 16, 1500
    n_log = n_pages * page // logical
    tdt = torch.float16 if dtype == torch.float16 else torch.bfloat16

    def vals(*shape):
        if case == "normal_f16":
            x = rng.standard_normal(shape)
        elif case == "wide_f16":  # subnormals (2^-24) up to 2^14
            x = rng.choice([-1, 1], shape) * np.exp2(rng.uniform(-24, 14, shape))
        elif case == "wide_bf16":
            x = rng.choice([-1, 1], shape) * np.exp2(rng.uniform(-120, 60, shape))
        else:  # products overflow fp32 -> err = inf -> every page scored exactly
            x = rng.standard_normal(shape) * 2.0**64
        return torch.from_numpy(x).to(tdt).double().numpy()

    stats = _stats_from(vals(n_log, d), vals(n_log, d))
    q = vals(rows, d)
    for k_pages in (4, 64, 700):
        pairs, exact, sel = _run(stats, q, dtype, page, logical, k_pages)
        approx, err = pairs[:, 0], pairs[:, 1]
        if k_pages == 64:
            finite = np.isfinite(err)
            assert np.all(np.abs(approx[finite] - exact[finite]) <= err[finite]), case
            if case == "normal_f16":  # the band stays small: the bound is not vacuous
                assert np.all(finite) and err.max() < 0.05 * np.abs(exact).max()
        assert sel == _oracle_sel(stats, q, page, logical, k_pages), (case, k_pages)
