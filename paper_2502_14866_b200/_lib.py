"""ctypes binding of the C ABI declared in ``include/sparsekv_b200.h``.

This is the only place the package touches native code.  The library is
loaded from the package directory; if it is missing, every compute entry
point raises -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

SK_OK, SK_EINVAL, SK_ECUDA, SK_EUNSUPPORTED = 0, -1, -2, -3
SK_F16, SK_BF16, SK_F32 = 0, 1, 2
SK_KIND_DENSE, SK_KIND_STREAMING = 0, 1
SK_DECODE_APPEND, SK_LAUNCH_PDL, SK_DECODE_SEL_READY = 1, 2, 4  # launch flags (sparsekv_b200.h)

LIB_PATH = os.environ.get("SK_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                       "libsparsekv_b200.so")

# every symbol include/sparsekv_b200.h declares (checked by tests/test_abi.py)
EXPORTS = ("sk_version", "sk_last_error", "sk_device_supported", "sk_slot_bytes", "sk_append_pages",
           "sk_append_token_layers",
           "sk_gather_pages", "sk_select_workspace", "sk_select_scores_offset", "sk_select_pages", "sk_score_pages",
           "sk_decode_workspace", "sk_decode_attn", "sk_prefill_attn", "sk_prefill_attn_paged")


class SkPool(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("head_dim", C.c_int32), ("page_size", C.c_int32),
                ("logical_page", C.c_int32), ("bits", C.c_int32), ("max_pages", C.c_int32),
                ("sink", C.c_int32), ("local", C.c_int32), ("slot_bytes", C.c_int64),
                ("arena", C.c_void_p), ("page_table", C.c_void_p), ("stats", C.c_void_p),
                ("staging", C.c_void_p), ("kind", C.c_void_p)]


class SkPrefillItem(C.Structure):
    _fields_ = [("head", C.c_int32), ("row0", C.c_int32), ("seg_begin", C.c_int32), ("seg_count", C.c_int32)]


_lib = None
_lock = threading.Lock()

_SIGS = {
    "sk_version": (C.c_char_p, []),
    "sk_last_error": (C.c_char_p, []),
    "sk_device_supported": (C.c_int, [C.c_int]),
    "sk_slot_bytes": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "sk_append_pages": (C.c_int, [C.POINTER(SkPool), C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                  C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "sk_append_token_layers": (C.c_int, [C.POINTER(SkPool), C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64,
                                         C.c_int64, C.POINTER(C.c_void_p), C.c_void_p]),
    "sk_gather_pages": (C.c_int, [C.POINTER(SkPool), C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64,
                                  C.c_int64, C.c_void_p]),
    "sk_select_workspace": (C.c_int64, [C.c_int32, C.c_int32]),
    "sk_select_scores_offset": (C.c_int64, [C.c_int32]),
    "sk_select_pages": (C.c_int, [C.POINTER(SkPool), C.c_int32, C.c_int32, C.c_void_p, C.c_int64, C.c_int64,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                  C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_uint32, C.c_void_p]),
    "sk_score_pages": (C.c_int, [C.POINTER(SkPool), C.c_int32, C.c_int32, C.c_void_p, C.c_int64, C.c_int64,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "sk_decode_workspace": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32]),
    "sk_decode_attn": (C.c_int, [C.POINTER(SkPool), C.c_int32, C.c_int32, C.c_void_p, C.c_int64, C.c_int64,
                                 C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_int32, C.c_void_p, C.c_float, C.c_void_p, C.c_int64, C.c_int64,
                                 C.c_int32, C.c_uint32, C.c_void_p, C.c_int64, C.c_void_p]),
    "sk_prefill_attn_paged": (C.c_int, [C.POINTER(SkPool), C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_float, C.c_void_p,
                                        C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sk_prefill_attn": (C.c_int, [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                  C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_float, C.c_void_p, C.c_int32,
                                  C.c_void_p, C.c_void_p, C.c_void_p]),
}


def load():
    """Load (once) and return the native library; raise if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"sparsekv-b200 CUDA library not built ({LIB_PATH}); "
                                   "run `python -c 'import __graft_entry__ as g; g.build()'`")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if hasattr(lib, "sk_debug_decode_stamps"):  # timing builds only
                lib.sk_debug_decode_stamps.restype = C.c_int
                lib.sk_debug_decode_stamps.argtypes = [C.c_void_p]
            _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc == SK_OK:
        return
    msg = load().sk_last_error().decode()
    if rc == SK_EINVAL:
        raise ValueError(msg)
    if rc == SK_EUNSUPPORTED:
        raise ValueError(f"unsupported on the B200 path: {msg}")
    raise RuntimeError(msg)


def version() -> str:
    return load().sk_version().decode()
