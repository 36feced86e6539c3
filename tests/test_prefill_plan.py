"""Block-mask parity of the K4 work plan (CPU): the (item, segment, flags)
lists the host builds for the prefill kernel must encode exactly the
reference's per-(head, query tile) tile schedules (attn.py:245-324,
engine.py:152-165; north_star: "block masks ... bit-exactly") and, with the
causal flag, exactly the reference's element-wise visible columns
(attn.py:315-319).  Decoding the plan back to masks needs no GPU."""

import numpy as np
import pytest

from oracle import sparsekv_oracle as O
from paper_2502_14866_b200 import Engine, EngineConfig, classify_heads
from paper_2502_14866_b200.attn import F_CAUSAL, F_MASKS, ITEM_ROWS, plan_from_segments, plan_generic, _segments_of


def decode_plan(plan, n_heads, n, s):
    """Per (head, 64-row query tile): visited 64-key blocks; and the element
    mask (row, column) the kernel applies."""
    tiles = {}
    elem = np.zeros((n_heads, n, s), bool)
    segs = plan.segs_np
    for head, row0, sb, sc in plan.items_np.tolist():
        for si in range(sb, sb + sc):
            first, word, mbase = segs[si].tolist()
            count, fl = word & 0xFFFFFF, word >> 24
            for i in range(count):
                blk = first + i
                for q in range(ITEM_ROWS // 64):
                    qt = row0 // 64 + q
                    if not fl & (1 << q) or qt * 64 >= n:
                        continue
                    tiles.setdefault((head, qt), []).append(blk)
                    for r in range(qt * 64, min(qt * 64 + 64, n)):
                        pos = r + (s - n)
                        for c in range(blk * 64, min(blk * 64 + 64, s)):
                            if (fl & F_CAUSAL) and c > pos:
                                continue
                            if fl & F_MASKS:
                                word_m = int(plan.masks_np[(mbase + i) * ITEM_ROWS + (r - row0)])
                                if not (word_m >> (c - blk * 64)) & 1:
                                    continue
                            elem[head, r, c] = True
    return tiles, elem


def reference_elem_mask(sched, n_heads, n, s, tq, tk):
    m = np.zeros((n_heads, n, s), bool)
    for (h, qt), tl in sched.items():
        for r in range(qt * tq, min(qt * tq + tq, n)):
            pos = r + (s - n)
            for t in tl:
                lo, hi = t * tk, min(t * tk + tk, s)
                m[h, r, lo:min(hi, pos + 1)] = True
    return m


@pytest.mark.parametrize("n,s,sink,local,sp", [(640, 640, 1, 4, 0.5), (200, 333, 1, 2, 0.5), (64, 64, 2, 1, 0.25),
                                               (1000, 1000, 1, 1, 0.75)])
def test_engine_plan_encodes_reference_schedules(n, s, sink, local, sp):
    h, h_kv = 8, 2
    gates = np.random.default_rng(n + s).uniform(0, 1, h).tolist()
    eng = Engine(EngineConfig(sink_blocks=sink, local_blocks=local, target_sparsity=sp),
                 classify_heads(gates, sp, sink, local), device="cpu")
    eng._group_size = h // h_kv
    plan = eng._plan(n, s)
    ref = O.OracleEngine(O.Config(sink_blocks=sink, local_blocks=local, target_sparsity=sp),
                         O.assign_roles(gates, sp, sink, local)).schedules(n, s)
    tiles, elem = decode_plan(plan, h, n, s)
    assert {k: sorted(v) for k, v in tiles.items()} == {k: sorted(v) for k, v in ref.items() if v}
    np.testing.assert_array_equal(elem, reference_elem_mask(ref, h, n, s, 64, 64))
    assert plan.visited.tolist() == [sum(len(ref[(hh, qt)]) for qt in range(-(-n // 64))) for hh in range(h)]


def test_random_schedules_and_generic_tiles():
    rng = np.random.default_rng(3)
    n, s, h = 300, 420, 4
    for tq, tk in ((64, 64), (32, 48), (100, 64)):
        n_qt, n_kt = -(-n // tq), -(-s // tk)
        sched = {}
        for hh in range(h):
            for qt in range(n_qt):
                diag = (s - n + min(qt * tq + tq, n) - 1) // tk
                pick = sorted(set(rng.choice(diag + 1, size=rng.integers(1, diag + 2), replace=False).tolist())
                              | {diag})
                sched[(hh, qt)] = pick
        if (tq, tk) == (64, 64):
            plan = plan_from_segments(lambda hh, qt: _segments_of(sched[(hh, qt)]), h, n, s)
        else:
            plan = plan_generic(sched, h, n, s, tq, tk)
        _, elem = decode_plan(plan, h, n, s)
        np.testing.assert_array_equal(elem, reference_elem_mask(sched, h, n, s, tq, tk), err_msg=f"{tq}x{tk}")
        assert n_kt > 0
