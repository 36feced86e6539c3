"""One small launch of every product kernel (K1 bulk + one-token append, K1b
gather, K2 select, K3 decode, K4 prefill), for compute-sanitizer
(tests/test_gpu_sanitizer.py).  Shapes are tiny so the instrumented run ends
in seconds; they still cross page boundaries, use GQA, both pools and the
reuse path."""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2502_14866_b200 as sk  # noqa: E402


def main() -> None:
    rng = np.random.default_rng(0)
    f = lambda *s: rng.standard_normal(s).astype(np.float16).astype(np.float32)  # noqa: E731
    n, h, h_kv, d = 300, 8, 2, 128
    gates = [0.9, 0.1, 0.8, 0.2, 0.05, 0.15, 0.12, 0.07]  # KV head 1 all-streaming (ring pool)
    cfg = sk.EngineConfig(quant_bits=4, budget_tokens=128, reuse_interval=2, sink_blocks=1, local_blocks=2)
    eng = sk.Engine(cfg, sk.classify_heads(gates, 0.5, 1, 2), device="cuda:0")
    eng.prefill(sk.Workload(f(n, h, d), f(n, h_kv, d), f(n, h_kv, d)))          # K4 + K1 bulk
    for _ in range(3):
        eng.decode_step(f(h, d), f(h_kv, d), f(h_kv, d))                          # K2, K3, K1 one-token
    eng.prefill_chunk(sk.Workload(f(70, h, d), f(70, h_kv, d), f(70, h_kv, d)))  # K1b + K4 + K1
    import torch
    torch.cuda.synchronize()
    print("sanitize probe ok")


if __name__ == "__main__":
    main()
