"""profiles/rNN_ncu_traffic.json from ncu reports (one launch each): DRAM
bytes and duration per kernel, read by bench.py's roofline.traffic.

    python tools/ncu_traffic.py OUT.json "source note" REPORT.ncu-rep ...
"""
import csv
import io
import json
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
         "msecond": 1e3, "ms": 1e3}


def read(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, d = rows[0], rows[1], rows[2]

    def val(name):
        i = h.index(name)
        return float(d[i].replace(",", "")) * SCALE.get(u[i], 1)

    name = d[h.index("Kernel Name")].split("(")[0].split("::")[-1].split("<")[0]
    return name, {"dram_read_bytes": val("dram__bytes_read.sum"), "dram_write_bytes": val("dram__bytes_write.sum"),
                  "duration_us": val("gpu__time_duration.sum"), "report": path.split("/")[-1]}


out = {"source": sys.argv[2], "kernels": {}}
for p in sys.argv[3:]:
    k, rec = read(p)
    out["kernels"][k] = rec
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps(out, indent=1))
