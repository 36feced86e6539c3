"""Per-CUDA-line warp-stall samples of an ncu report (source page): the
lines with the most samples and their share.
Usage: python tools/ncu_lines.py REPORT.ncu-rep [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r][0]
h = rows[hi]
st = h.index("Warp Stall Sampling (All Samples)")


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


lines = [(int(r[0]), r[1], num(r[st])) for r in rows[hi + 1:] if len(r) == len(h) and r[0].isdigit()]
tot = sum(x[2] for x in lines)
print(f"total samples {tot:.0f}")
for ln, src, v in sorted(lines, key=lambda x: -x[2])[:top]:
    print(f"{v:7.0f} {100 * v / tot:5.1f}%  L{ln:<5d} {src.strip()[:100]}")
