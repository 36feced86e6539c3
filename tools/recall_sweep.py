"""Selection-recall sweep at 128k on the B200 selector (
the reference's sweeps.clustered_recall / C06-C07 at real context length).

cfg2 geometry per KV head (D 128, 4 query rows), 32 device-generated trials
per point, needle and clustered_needles workloads at two margins, budgets
512..4096 tokens, three paging schemes + the exact-score oracle.  One JSON
line per (kind, margin)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2502_14866_b200 import recall as R
from paper_2502_14866_b200 import workloads as W


def main():
    out = open(os.environ["SK_SWEEP_OUT"], "w") if os.environ.get("SK_SWEEP_OUT") else None
    budgets = (512, 1024, 2048, 4096)
    for kind, span in ((W.NEEDLE, 1), (W.CLUSTERED, 4)):
        for margin in (0.05, 1.0):
            t0 = time.time()
            batch = W.gen_needles_device(kind, 32, 131072, 128, 4, margin=margin, cluster_span=span, seed=1,
                                         device="cuda:0")
            res = R.batch_recall(batch, budgets)
            torch.cuda.synchronize()
            rec = {"kind": kind, "context": 131072, "head_dim": 128, "group_rows": 4, "trials": 32,
                   "cluster_span": span, "margin": margin, "recall": {str(b): res[b] for b in budgets},
                   "wall_s": round(time.time() - t0, 2)}
            line = json.dumps(rec)
            print(line, flush=True)
            if out:
                out.write(line + "\n")
            del batch
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
