#!/bin/bash
# device loop vs host loop A/B on c1 / c2 / c4 (PDL, gate block)
mkdir -p gpurun_out
for c in c2 c1; do
timeout 900 python tools/loop_ab.py --config $c --steps 5 PINT_DEVICE_LOOP=0 PINT_DEVICE_LOOP=1 "PINT_DEVICE_LOOP=0 PINT_PDL=0" "PINT_DEVICE_LOOP=1 PINT_PDL=0" "PINT_DEVICE_LOOP=1 PINT_GATE=2" "PINT_DEVICE_LOOP=1 PINT_GATE=4" >> gpurun_out/b_ab.jsonl 2>> gpurun_out/b_ab.err
done
timeout 600 python tools/loop_ab.py --config c1 --slices 1 --steps 3 PINT_DEVICE_LOOP=0 PINT_DEVICE_LOOP=1 "PINT_DEVICE_LOOP=1 PINT_GATE=4" >> gpurun_out/b_ab.jsonl 2>> gpurun_out/b_ab.err
timeout 900 python tools/loop_ab.py --config c4 --steps 2 PINT_DEVICE_LOOP=0 PINT_DEVICE_LOOP=1 >> gpurun_out/b_ab.jsonl 2>> gpurun_out/b_ab.err
