"""pytest plugin: run the reference's own hot-path tests against
paper_2502_14866_b200 by aliasing ``sparsekv`` (and its submodules) to this
package -- the module swap a sparsekv user makes.

Known deviations are marked xfail here, each with its reason; everything
else must pass unmodified.  The reasons fall into three groups:

* WIDE: the test feeds fp64 values that fp16 (the device dtype) cannot hold
  and checks page stats / codes / scores exactly.  The B200 boundary refuses
  such inputs (ValueError, paper_2502_14866_b200.allow_input_rounding)
  instead of rounding them silently.
* TOL: the test compares attention at 1e-10..1e-12 of an fp64 result; the
  B200 path computes attention on fp16 tensor cores (north_star tolerance
  2e-2 / cosine 0.9999, met by tests/test_gpu_parity.py).
* DTYPE: the test checks that outputs carry the input's float64/float32
  dtype bit for bit from an fp64 computation.
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

WIDE = "fp64 inputs not exact in fp16: refused at the B200 boundary instead of silently rounded"
TOL = "fp16 tensor-core attention: north_star tolerance (2e-2 / cos 0.9999), not the fp64 1e-10 bound"
DTYPE = "outputs are computed in fp16 on the device, not in the fp64 input dtype"

# test name (file::test, without parametrisation) -> reason; filled from the
# GPU run of tests/test_gpu_reference_suite.py
XFAIL: dict = {}


def pytest_collection_modifyitems(config, items):
    for item in items:
        key = item.nodeid.split("/")[-1]
        reason = XFAIL.get(key) or XFAIL.get(key.split("[")[0])
        if reason:
            item.add_marker(pytest.mark.xfail(reason=reason, strict=False))
