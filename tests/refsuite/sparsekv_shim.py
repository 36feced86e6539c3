"""pytest plugin: run the reference's own hot-path tests against
paper_2502_14866_b200 by aliasing ``sparsekv`` (and its submodules) to this
package -- the module swap a sparsekv user makes.

Known deviations are marked xfail here, each with its reason; everything
else must pass unmodified.  The reasons fall into three groups:

* WIDE: the test feeds fp64 values that fp16 (the device dtype) cannot hold
  and checks page stats / codes / scores against them exactly.  The product
  refuses such inputs by default (ValueError); this shim opts in to rounding
  (allow_input_rounding), so these tests see fp16-rounded stats.
* TOL: the test compares attention at 1e-10..1e-12 of an fp64 result; the
  B200 path computes attention on fp16 tensor cores (north_star tolerance
  2e-2 / cosine 0.9999, met by tests/test_gpu_parity.py).

The same properties hold on the B200 path at its own precision: attention
within the north_star tolerance of the reference's fp32 output, and stats /
codes / selections bit-exact for fp16-valued inputs (tests/test_gpu_parity.py,
test_gpu_cfg1_golden.py against the reference's own runs).
"""

from __future__ import annotations

import importlib
import sys

import pytest

SUBMODULES = ("attn", "cache", "engine", "heads", "ledger", "selector", "workloads")


def _alias() -> None:
    pkg = importlib.import_module("paper_2502_14866_b200")
    sys.modules["sparsekv"] = pkg
    for name in SUBMODULES:
        sys.modules[f"sparsekv.{name}"] = importlib.import_module(f"paper_2502_14866_b200.{name}")


_alias()
# A sparsekv user hands the reference fp64 arrays; the device stores fp16.
# The shim opts in to rounding (paper_2502_14866_b200.allow_input_rounding,
# off by default: the product refuses inexact inputs) so the behavioural
# tests run; the tests whose assertions need fp64 storage are the xfails.
importlib.import_module("paper_2502_14866_b200").allow_input_rounding(True)

WIDE = "fp64 inputs are stored in fp16 on the device: exact-fp64 stats / codes / scores are not reproduced"
TOL = "fp16 tensor-core attention: north_star tolerance (2e-2 / cos 0.9999), not the fp64 1e-10 bound"

# test name (file::test, without parametrisation) -> reason, from the GPU run
# of tests/test_gpu_reference_suite.py (115 tests: 100 pass, these 15 xfail)
XFAIL: dict = {
    # attention compared with an fp64 result at 1e-10..1e-12
    "test_attn.py::test_full_schedule_matches_reference": TOL,
    "test_attn.py::test_random_partial_schedules_match_restricted_oracle": TOL,
    "test_attn.py::test_last_tile_only_equals_restricted_oracle": TOL,
    "test_engine.py::test_all_retrieval_prefill_matches_reference": TOL,
    "test_engine.py::test_streaming_prefill_output_matches_masked_oracle": TOL,
    "test_engine.py::test_full_budget_decode_matches_one_row_reference": TOL,
    "test_engine.py::test_mixed_group_streaming_head_reads_the_dense_pool": TOL,
    "test_engine.py::test_stage_consistency_decode_equals_longer_prefill": TOL,
    # page stats / codes / raw pages / scores compared with the fp64 inputs exactly
    "test_cache.py::test_reconstruction_error_within_half_scale": WIDE,
    "test_cache.py::test_bits_none_stores_raw": WIDE,
    "test_cache.py::test_single_token_stats_collapse_to_the_key": WIDE,
    "test_cache.py::test_stats_match_bruteforce_minmax_over_long_stream": WIDE,
    "test_cache.py::test_bounding_box_soundness_over_a_million_samples": WIDE,
    "test_cache.py::test_lookup_examples_and_roundtrip": WIDE,
    "test_selector.py::test_score_pages_matches_scalar_path": WIDE,
}


def pytest_collection_modifyitems(config, items):
    for item in items:
        key = item.nodeid.split("/")[-1]
        reason = XFAIL.get(key) or XFAIL.get(key.split("[")[0])
        if reason:
            item.add_marker(pytest.mark.xfail(reason=reason, strict=False))
