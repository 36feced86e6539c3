timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b.csv python tools/profile_batched.py > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_b.csv | grep -v "at::"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_kernel -c 1 -o gpurun_out/ncu_b_select python tools/profile_batched.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -c 1 -o gpurun_out/ncu_b_decode python tools/profile_batched.py > /dev/null 2>&1
