"""K2 phase B's value-linear histogram passes (csrc/select.cu, topk_filtered)
on score distributions chosen to stress them: outliers that squeeze every other
page into one bin (a second and third pass must split it), far-apart clusters
with the K-th score inside the dense one, negative-only scores, exact ties at
the K-th score (broken by page index, selector.py:106) next to an outlier, and
scores packed into a range narrower than the error band.  The selection must
equal the oracle's fp64 (score desc, index asc) ranking (selector.py:81-108)."""

import numpy as np
import pytest
import torch

from test_gpu_select_bound import _oracle_sel, _run

pytestmark = pytest.mark.gpu

PAGE, LOGICAL, D, ROWS = 64, 16, 128, 2


def _scores(case, n, rng):
    if case == "outlier":
        s = rng.standard_normal(n)
        s[n // 3] = 4000.0
    elif case == "three_outliers_ties":
        s = np.round(rng.standard_normal(n) * 4) / 4  # many exact ties
        s[[5, n // 2, n - 7]] = [9000.0, -9000.0, 7000.0]
    elif case == "clusters":
        s = np.where(rng.random(n) < 0.9, rng.standard_normal(n) * 0.01, 500.0 + rng.standard_normal(n) * 0.01)
    elif case == "negative":
        s = -50.0 - np.abs(rng.standard_normal(n)) * 10
    elif case == "narrow":
        s = 3.0 + rng.standard_normal(n) * 1e-3
    else:
        raise ValueError(case)
    return s


@pytest.mark.parametrize("case", ["outlier", "three_outliers_ties", "clusters", "negative", "narrow"])
@pytest.mark.parametrize("n_pages", [1000, 2048])
def test_value_linear_passes_against_oracle(case, n_pages):
    rng = np.random.default_rng(sum(map(ord, case)) + n_pages)
    s = _scores(case, n_pages, rng)
    lp = PAGE // LOGICAL
    # q = ones: a logical page whose k_min = k_max = v (all channels) scores D * v;
    # the page's first logical page carries the score, the others sit below it
    v = torch.from_numpy(s / D).to(torch.float16).double().numpy()
    stats = np.empty((n_pages * lp, 2, D))
    for i in range(n_pages):
        for j in range(lp):
            x = v[i] if j == 0 else torch.tensor(v[i] - abs(v[i]) - 1.0).half().double().item()
            stats[i * lp + j, :, :] = x
    q = np.ones((ROWS, D))
    for k_pages in (8, 64, n_pages // 4):
        _, _, sel = _run(stats, q, torch.float16, PAGE, LOGICAL, k_pages)
        assert sel == _oracle_sel(stats, q, PAGE, LOGICAL, k_pages), (case, n_pages, k_pages)
