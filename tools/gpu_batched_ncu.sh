#!/usr/bin/env bash
# cfg4 batched decode: per-kernel duration / DRAM / issue (ncu launch list, 2 layers)
cd "$(dirname "$0")/.."
SK_LAYERS=8 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__grid_size \
  --clock-control none --csv --log-file gpurun_out/batched_launches.csv python tools/batched_probe.py > gpurun_out/batched_ncu.log 2>&1
python tools/launch_metrics.py gpurun_out/batched_launches.csv
