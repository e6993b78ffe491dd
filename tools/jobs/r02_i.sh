#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/loop_ab.py --config c3 --steps 2 PINT_A32C=0 PINT_A32C=1 > gpurun_out/i_ab.jsonl 2> gpurun_out/i_ab.err
timeout 900 python tools/loop_ab.py --config c4 --steps 2 PINT_A32C=0 PINT_A32C=1 >> gpurun_out/i_ab.jsonl 2>> gpurun_out/i_ab.err
timeout 900 python tools/loop_ab.py --config c2 --steps 5 PINT_A32C=0 PINT_A32C=1 >> gpurun_out/i_ab.jsonl 2>> gpurun_out/i_ab.err
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/i_gpu.log 2>&1
timeout 600 python tools/parareal_analysis.py order --config c1 > gpurun_out/i_order.jsonl 2>&1
timeout 900 python tools/parareal_analysis.py fields --config c1 > gpurun_out/i_fields_c1.jsonl 2>&1
