"""K3 over pages whose per-channel ranges span several orders of magnitude.

K3 feeds the stored codes to the tensor cores as fp16 subnormals (n * 2^-24,
the odd nibble slots as 16 n * 2^-24 with the matching 1/16 on the B operand)
and undoes the 2^-24 with the page scale (decode.cu, nib2h / kCodeUnscale).
These cases pin that arithmetic against the oracle's dequantise-then-attend
(reference engine.py:257-285, cache.py:97-102) where it is most exposed: tiny
and large channel scales in one page, constant channels (scale 0), every code
width K3 decodes (nibbles for 2/3/4 bits, bytes for 8), fp16 and bf16 pools.
Outputs are compared relative to the value scale, with the parity tolerance
of tests/test_gpu_parity.py."""

import numpy as np
import pytest
import torch

import paper_2502_14866_b200 as sk
from oracle import sparsekv_oracle as O

pytestmark = pytest.mark.gpu

ATOL, MIN_COS = 2e-2, 0.9999


def _rounded(x, dtype):
    return torch.from_numpy(x.astype(np.float32)).to(dtype).float().numpy()


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16], ids=["f16", "bf16"])
@pytest.mark.parametrize("bits", [4, 8, 2])
@pytest.mark.parametrize("scale", [1e-3, 1.0, 200.0])
def test_decode_wide_channel_ranges_vs_oracle(dtype, bits, scale):
    rng = np.random.default_rng(int(scale * 1000) % 997 + bits)
    s, h, h_kv, d = 900, 8, 2, 128
    gates = [0.9, 0.1, 0.8, 0.2, 0.85, 0.15, 0.95, 0.05]
    # per-channel magnitudes over 3 decades, a few constant channels
    ch = scale * 10.0 ** rng.uniform(-3, 0, d)
    k = rng.standard_normal((s, h_kv, d)) * ch
    v = rng.standard_normal((s, h_kv, d)) * ch
    k[:, :, :3] = 0.25 * scale
    v[:, :, 5:7] = -0.5 * scale
    k, v = _rounded(k, dtype), _rounded(v, dtype)
    cfg = dict(quant_bits=bits, budget_tokens=320, reuse_interval=2, local_blocks=2)
    prof = sk.classify_heads(gates, 0.5, 1, 2)
    eng = sk.Engine(sk.EngineConfig(**cfg), prof, device="cuda:0", dtype=dtype)
    eng.load_context(k, v)
    ref = O.OracleEngine(O.Config(**cfg), O.assign_roles(gates, 0.5, 1, 2))
    ref.load_context(k, v)
    for t in range(6):
        qn = _rounded(rng.standard_normal((h, d)) / np.sqrt(max(scale, 1e-3)) * (0.05 if scale > 10 else 1.0), dtype)
        kn = _rounded(rng.standard_normal((h_kv, d)) * ch, dtype)
        vn = _rounded(rng.standard_normal((h_kv, d)) * ch, dtype)
        res = eng.decode_step(qn, kn, vn)
        rr = ref.decode_step(qn, kn, vn)
        assert [tuple(tb.positions) for tb in res.index_tables] == rr.tables, f"step {t}"
        out = np.asarray(res.output, np.float64) / scale
        want = np.asarray(rr.output, np.float64) / scale
        err = np.abs(out - want).max()
        assert err <= ATOL, f"step {t}: max-abs / scale {err:.3e}"
        cos = (out * want).sum(-1) / (np.linalg.norm(out, axis=-1) * np.linalg.norm(want, axis=-1) + 1e-30)
        assert cos.min() >= MIN_COS, f"step {t}: min cosine {cos.min():.7f}"
