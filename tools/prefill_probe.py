"""K4 alone on one 128k-context layer (cfg2 shapes, balanced gates): mean
launch time over `reps` CUDA-event-timed launches, TFLOP/s on the ledger
count, and the SM clock sampled during the launches (nvidia-smi).  Loads
whatever library SK_LIB_PATH points at (A/B experiments)."""
import math
import os
import subprocess
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2502_14866_b200 as sk
from paper_2502_14866_b200.attn import run_prefill

ctx = int(os.environ.get("SK_CTX", 131072))
reps = int(os.environ.get("SK_REPS", 6))
H, HKV, D = 32, 8, 128
gates = [0.9 - 0.001 * h if h % 4 < 2 else 0.1 + 0.001 * h for h in range(H)]
eng = sk.Engine(sk.EngineConfig(quant_bits=4, local_blocks=4), sk.classify_heads(gates, 0.5, 1, 4), device="cuda:0")
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn((ctx, H, D), generator=g, device="cuda", dtype=torch.float16)
k = torch.randn((ctx, HKV, D), generator=g, device="cuda", dtype=torch.float16)
v = torch.randn((ctx, HKV, D), generator=g, device="cuda", dtype=torch.float16)
eng._group_size = H // HKV
plan = eng._plan(ctx, ctx)
flop = int(plan.visited.sum()) * 4 * 64 * 64 * D
for _ in range(2):
    run_prefill(q, k, v, plan, 1 / math.sqrt(D))
torch.cuda.synchronize()
clk, stop = [], threading.Event()


def sample():
    while not stop.is_set():
        out = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True).stdout.strip()
        if out.isdigit():
            clk.append(int(out))
        stop.wait(0.1)


th = threading.Thread(target=sample, daemon=True)
th.start()
ts = []
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run_prefill(q, k, v, plan, 1 / math.sqrt(D))
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
stop.set()
th.join()
ms = sum(ts) / len(ts)
clk.sort()
print(f"{os.path.basename(os.environ.get('SK_LIB_PATH', 'default'))}: K4 {ms:.2f} ms/layer  "
      f"{flop / ms / 1e9:.0f} TFLOP/s  frac {flop / ms / 1e9 / 1654.2:.3f}  sm_mhz median "
      f"{clk[len(clk) // 2] if clk else None}  min {clk[0] if clk else None}")
