"""CPU-side checks of the native boundary: the library builds for sm_100a,
loads, and exports every symbol include/sparsekv_b200.h declares (no
compute without a GPU)."""

import ctypes
import os
import re

import pytest

from paper_2502_14866_b200 import _build, _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        _build.build(verbose=False)
    return ctypes.CDLL(_lib.LIB_PATH)


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "sparsekv_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(sk_[a-z_]+)\s*\(", hdr)))


def test_header_declares_the_binding_exports():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_pure_host_entry_points(lib):
    L = _lib.load()
    assert b"sm_100a" in L.sk_version()
    assert L.sk_slot_bytes(128, 64, 4, 0) == 9216          # KV4 page: 8 KB codes + 1 KB bounds
    assert L.sk_slot_bytes(128, 64, 0, 0) == 32768         # fp16 page
    assert L.sk_select_workspace(8, 2048) >= 8 * 2048 * 16
    off = L.sk_select_scores_offset(8)
    assert off >= 8 * 4 and off % 256 == 0                 # tickets first, scores 256-B aligned after them
    assert L.sk_select_workspace(8, 2048) == off + 8 * 2048 * 16


def test_sass_contains_tcgen05_and_tma(lib):
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([cuobjdump, "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass or "UTCQMMA" in sass     # tcgen05.mma (prefill)
    assert "UTMALDG" in sass                          # TMA loads (prefill)
    assert "LDTM" in sass                             # tcgen05.ld (TMEM -> registers)
    assert "HMMA" in sass                             # mma.sync (decode on quantised pages)
