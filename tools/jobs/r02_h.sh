#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/elem_ab.py > gpurun_out/h_elem_ab.jsonl 2> gpurun_out/h_elem_ab.err
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/h_gpu.log 2>&1
timeout 900 python tools/loop_ab.py --config c3 --steps 2 PINT_DEVICE_LOOP=1 PINT_ELEM=old >> gpurun_out/h_ab.jsonl 2>> gpurun_out/h_ab.err
timeout 900 python tools/loop_ab.py --config c4 --steps 2 PINT_DEVICE_LOOP=1 PINT_ELEM=old >> gpurun_out/h_ab.jsonl 2>> gpurun_out/h_ab.err
