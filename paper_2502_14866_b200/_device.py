"""Device/dtype plumbing shared by the host modules (PyTorch is plumbing here:
device memory, streams; all hot-path compute is in the C-ABI library)."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

DEFAULT_DTYPE = torch.float16
_checked: set = set()


def device_of(device=None) -> torch.device:
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None
    if device is None:
        raise RuntimeError("sparsekv-b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback")
    device = torch.device(device)
    if device.type != "cuda":
        raise RuntimeError("sparsekv-b200 runs on CUDA devices only; there is no CPU fallback")
    idx = device.index if device.index is not None else torch.cuda.current_device()
    if idx not in _checked:
        lib = _lib.load()
        if not lib.sk_device_supported(idx):
            raise RuntimeError(f"cuda:{idx} is not an sm_100 (B200) device; this build targets sm_100a only")
        _checked.add(idx)
    return torch.device("cuda", idx)


def sk_dtype(dtype: torch.dtype) -> int:
    if dtype == torch.float16:
        return _lib.SK_F16
    if dtype == torch.bfloat16:
        return _lib.SK_BF16
    raise ValueError(f"device dtype must be float16 or bfloat16, got {dtype}")


def padded_dim(d: int) -> int:
    if d < 1:
        raise ValueError("head_dim must be positive")
    if d > 128:
        raise ValueError(f"head_dim {d} > 128 is not supported on the B200 path")
    return 64 if d <= 64 else 128


def is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


_ALLOW_ROUNDING = False


def allow_input_rounding(flag: bool = True) -> None:
    """Opt in to rounding wider inputs (fp32/fp64) to the device dtype.

    The reference computes in its input dtype (attn.py:28-30).  The B200 path
    stores pages, statistics and queries in fp16/bf16, so its page stats,
    codes and selections equal the reference's only for inputs the device
    dtype represents exactly; by default any other input is refused with a
    ValueError instead of being rounded silently."""
    global _ALLOW_ROUNDING
    _ALLOW_ROUNDING = bool(flag)


class rounding_allowed:
    """Context manager: allow_input_rounding(True) inside, the previous
    policy restored on exit (for harness code that only counts tiles)."""

    def __enter__(self):
        self._prev = _ALLOW_ROUNDING
        allow_input_rounding(True)
        return self

    def __exit__(self, *exc):
        allow_input_rounding(self._prev)
        return False


def _check_exact(src: torch.Tensor, dst: torch.Tensor) -> None:
    """src (wide, on the device) == dst (device dtype) element for element;
    NaN passes here so the callers' finiteness checks keep their messages."""
    back = dst.to(src.dtype)
    bad = ~((back == src) | torch.isnan(src))
    if bool(bad.any()):
        i = int(bad.flatten().nonzero()[0])
        raise ValueError(f"input value {src.flatten()[i].item()!r} is not exactly representable in {dst.dtype} "
                         f"(the device dtype); cast the inputs to {dst.dtype} first, or call "
                         f"paper_2502_14866_b200.allow_input_rounding(True) to accept rounded page stats")


def to_device(x, dtype: torch.dtype, device: torch.device, pad_to: int | None = None) -> torch.Tensor:
    """numpy / torch -> contiguous device tensor of `dtype`, last dim zero-padded.
    Wider floating inputs must be exact in `dtype` (see allow_input_rounding)."""
    t = x if is_torch(x) else torch.from_numpy(np.ascontiguousarray(x))
    if t.dtype != dtype and t.is_floating_point() and not _ALLOW_ROUNDING:
        wide = t.to(device=device, non_blocking=True)
        t = wide.to(dtype)
        _check_exact(wide, t)
    else:
        t = t.to(device=device, dtype=dtype, non_blocking=True)
    if pad_to is not None and t.shape[-1] != pad_to:
        t = torch.nn.functional.pad(t, (0, pad_to - t.shape[-1]))
    return t.contiguous()


def exact_cast(t: torch.Tensor, dtype: torch.dtype) -> torch.Tensor:
    """t.to(dtype), refusing values `dtype` cannot hold exactly (unless rounding is allowed)."""
    out = t.to(dtype)
    if t.dtype != dtype and t.is_floating_point() and not _ALLOW_ROUNDING:
        _check_exact(t, out)
    return out


def h2d(a, device: torch.device, dtype=None) -> torch.Tensor:
    """Small host array -> device without a blocking pageable copy (pinned,
    caching host allocator, stream-ordered)."""
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.pin_memory().to(device, non_blocking=True)


def stream_ptr(device: torch.device):
    return torch.cuda.current_stream(device).cuda_stream


def to_output(t: torch.Tensor, like, np_dtype=None):
    """Return in the caller's flavour: torch in -> torch out, numpy in -> numpy out."""
    if is_torch(like):
        return t
    out = t.float().cpu().numpy()
    return out.astype(np_dtype) if np_dtype is not None else out


def all_finite(t: torch.Tensor) -> torch.Tensor:
    """Device bool scalar: no NaN/inf in t.  One read of t (max-norm; NaN and
    inf propagate through it), no full-size temporaries."""
    if not t.is_floating_point():
        return torch.ones((), dtype=torch.bool, device=t.device)
    return torch.isfinite(torch.linalg.vector_norm(t, float("inf")))
