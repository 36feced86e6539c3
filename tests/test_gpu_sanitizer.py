"""compute-sanitizer over one small launch of every product kernel
(tools/sanitize_probe.py): memcheck (out-of-bounds / misaligned accesses),
racecheck (shared-memory hazards: K2's bulk-copy slots, K3's DSMEM inboxes,
K4's smem rings), synccheck (barrier misuse) and initcheck (reads of
uninitialised device memory).  SURVEY.md 5."""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.skipif(not os.path.exists(SAN), reason="compute-sanitizer not installed")
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_kernels_are_clean_under_compute_sanitizer(tool):
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--target-processes", "all",
           "--kernel-name", "regex:(append|gather|select|decode|prefill)",
           sys.executable, os.path.join(ROOT, "tools", "sanitize_probe.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    out = res.stdout + res.stderr
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"sanitizer_{tool}.log"), "w") as fp:
        fp.write(out)
    assert res.returncode == 0 and "sanitize probe ok" in out, out[-5000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-5000:]
