#!/bin/bash
# closing c3 launch list (time + DRAM bytes) at the final tree
mkdir -p gpurun_out
export PINT_DEVICE_LOOP=0
timeout 600 python tools/profile_step.py --config c3 --steps 2 > gpurun_out/bl_plain_c3.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --nvtx --nvtx-include "prof/" --csv --log-file gpurun_out/bl_launches_c3.csv \
  python tools/profile_step.py --config c3 --steps 2 > gpurun_out/bl_ncu_launch_c3.log 2>&1
gzip -f gpurun_out/bl_launches_c3.csv
true
