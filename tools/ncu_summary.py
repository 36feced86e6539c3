"""Summarise ncu --set full reports (.ncu-rep) into a markdown table.

    python tools/ncu_summary.py gpurun_out/ncu_*.ncu-rep > profiles/rNN_ncu_summary.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("duration us", "gpu__time_duration.sum", 1e-3),
    ("DRAM read MB", "dram__bytes_read.sum", 1e-6),
    ("DRAM write MB", "dram__bytes_write.sum", 1e-6),
    ("DRAM % peak", "dram__bytes_read.sum.pct_of_peak_sustained_elapsed", 1),
    ("tensor pipe %", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    ("issue active %", "sm__issue_active.avg.pct_of_peak_sustained_elapsed", 1),
    ("ALU pipe %", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
    ("FMA pipe %", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
    ("XU (MUFU) pipe %", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1),
    ("FP64 pipe %", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1),
    ("achieved occupancy %", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("registers/thread", "launch__registers_per_thread", 1),
    ("grid", "launch__grid_size", 1),
    ("block", "launch__block_size", 1),
    ("smem wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1),
    ("smem bank-conflict wavefronts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
]
UNIT_SCALE = {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
              "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    out = []
    for data in rows[2:]:
        rec = {"kernel": data[h.index("Kernel Name")].split("(")[0][:60]}
        for label, name, scale in METRICS:
            if name not in h:
                rec[label] = "-"
                continue
            i = h.index(name)
            try:
                val = float(data[i].replace(",", ""))
            except ValueError:
                rec[label] = data[i]
                continue
            base = UNIT_SCALE.get(u[i], 1)
            if label.endswith(" us"):
                val = val * base / 1e3
            elif label.endswith(" MB"):
                val = val * base / 1e6
            rec[label] = f"{val:.4g}"
        out.append(rec)
    return out


def main():
    recs = []
    for p in sys.argv[1:]:
        recs += [(p, r) for r in summarise(p)]
    labels = ["kernel"] + [m[0] for m in METRICS]
    print("| report | " + " | ".join(labels) + " |")
    print("|" + "---|" * (len(labels) + 1))
    for p, r in recs:
        print(f"| {p.split('/')[-1]} | " + " | ".join(str(r.get(k, "-")) for k in labels) + " |")


if __name__ == "__main__":
    main()
