#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/loop_ab.py --config c1 --slices 1 --steps 3 PINT_DEVICE_LOOP=0 "PINT_GATE=4" "PINT_GATE=8" "PINT_GATE=30" "PINT_GATE=4 PINT_GATE0=4" "PINT_GATE=4 PINT_GATE0=8" >> gpurun_out/c_ab.jsonl 2>> gpurun_out/c_ab.err
timeout 900 python tools/loop_ab.py --config c2 --steps 5 PINT_DEVICE_LOOP=0 "PINT_GATE=4" "PINT_GATE=8" "PINT_GATE=4 PINT_GATE0=4" "PINT_GATE=4 PINT_GATE0=8" >> gpurun_out/c_ab.jsonl 2>> gpurun_out/c_ab.err
timeout 900 python tools/loop_ab.py --config c3 --steps 2 PINT_DEVICE_LOOP=0 "PINT_GATE=4" "PINT_GATE=4 PINT_GATE0=8" >> gpurun_out/c_ab.jsonl 2>> gpurun_out/c_ab.err
for v in "PINT_DEVICE_LOOP=0" "PINT_GATE=4" "PINT_GATE=4 PINT_GATE0=4"; do
  env $v timeout 600 python tools/parareal_run.py --config c1 | sed "s/^/$v /" >> gpurun_out/c_parareal.log 2>&1
done
