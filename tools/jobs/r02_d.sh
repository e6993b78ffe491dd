#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_device_loop.py -x -q > gpurun_out/d_loop.log 2>&1
timeout 900 python tools/loop_ab.py --config c1 --slices 1 --steps 3 PINT_DEVICE_LOOP=0 PINT_DEVICE_LOOP=1 "PINT_GATE0=4" "PINT_GATE0=12" >> gpurun_out/d_ab.jsonl 2>> gpurun_out/d_ab.err
timeout 900 python tools/loop_ab.py --config c1 --steps 5 PINT_DEVICE_LOOP=0 PINT_DEVICE_LOOP=1 >> gpurun_out/d_ab.jsonl 2>> gpurun_out/d_ab.err
timeout 900 python tools/loop_ab.py --config c2 --steps 5 PINT_DEVICE_LOOP=0 PINT_DEVICE_LOOP=1 "PINT_GATE0=12" "PINT_GATE=2" >> gpurun_out/d_ab.jsonl 2>> gpurun_out/d_ab.err
timeout 900 python tools/loop_ab.py --config c4 --steps 2 PINT_DEVICE_LOOP=0 PINT_DEVICE_LOOP=1 >> gpurun_out/d_ab.jsonl 2>> gpurun_out/d_ab.err
for v in "PINT_DEVICE_LOOP=0" "PINT_DEVICE_LOOP=1"; do
  env $v timeout 600 python tools/parareal_run.py --config c1 | sed "s/^/$v /" >> gpurun_out/d_parareal.log 2>&1
done
