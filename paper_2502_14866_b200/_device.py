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


def to_device(x, dtype: torch.dtype, device: torch.device, pad_to: int | None = None) -> torch.Tensor:
    """numpy / torch -> contiguous device tensor of `dtype`, last dim zero-padded."""
    t = x if is_torch(x) else torch.from_numpy(np.ascontiguousarray(x))
    t = t.to(device=device, dtype=dtype, non_blocking=True)
    if pad_to is not None and t.shape[-1] != pad_to:
        t = torch.nn.functional.pad(t, (0, pad_to - t.shape[-1]))
    return t.contiguous()


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
