#!/bin/bash
# configs parity tests; ncu launch list (time + DRAM bytes) of a 2-step c3 window (host loop: same kernels)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_configs.py -q > gpurun_out/e_configs.log 2>&1
export PINT_DEVICE_LOOP=0
timeout 600 python tools/profile_step.py --config c3 --steps 2 > gpurun_out/e_plain.log 2>&1 && \
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --nvtx --nvtx-include "prof/" --csv --log-file gpurun_out/e_launches_c3.csv python tools/profile_step.py --config c3 --steps 2 > gpurun_out/e_ncu.log 2>&1
true
