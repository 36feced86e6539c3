"""The reference's own hot-path test files (pkg/tests/test_{attn,cache,
selector,heads,engine,workloads}.py), run unmodified against this package
through an import alias (tests/refsuite/sparsekv_shim.py): the drop-in
check of SURVEY.md 8(c) item 3.  tools/install_reference.sh copies the suite
next to the reference install (baseline/_ref, which travels to the GPU box);
the xfails are listed, with reasons, in the shim."""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "baseline", "_ref", "sparsekv_tests")
FILES = ["test_attn.py", "test_cache.py", "test_selector.py", "test_heads.py", "test_engine.py",
         "test_workloads.py"]


@pytest.mark.skipif(not os.path.isdir(SUITE), reason="reference suite not installed (tools/install_reference.sh)")
def test_reference_suite_against_this_package():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests", "refsuite"), ROOT])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    # A fixed hypothesis seed: the reference's own property test
    # test_partition_is_invariant_under_monotone_transforms (test_heads.py:45)
    # fails for the unmodified reference too on some random draws -- x / (1 + x)
    # maps gates 0.9989999999999999 and 0.999 to one float, and the tie then
    # goes to the lower head index -- so unseeded runs are flaky for both.
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "sparsekv_shim", "-p", "no:cacheprovider", "-rxf",
           "--hypothesis-seed=0", "--rootdir", SUITE, "-o", "addopts=", *[os.path.join(SUITE, f) for f in FILES]]
    res = subprocess.run(cmd, cwd=SUITE, env=env, capture_output=True, text=True, timeout=1800)
    out = res.stdout + res.stderr
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "reference_suite.log"), "w") as fp:
        fp.write(out)
    summary = out.strip().splitlines()[-1] if out.strip() else ""
    counts = {k: int(v) for v, k in re.findall(r"(\d+) (passed|failed|xfailed|xpassed|errors?)", summary)}
    assert res.returncode == 0 and not counts.get("failed") and not counts.get("error"), out[-6000:]
    assert counts.get("passed", 0) >= 60, summary
