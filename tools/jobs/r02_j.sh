#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/parareal_analysis.py order --config c1 --theta0 0 > gpurun_out/j_order_cn.jsonl 2>&1
timeout 600 python tools/parareal_analysis.py order --config c1 --t-final 0.05 --steps 0.002 0.001 0.0005 0.00025 > gpurun_out/j_order_short.jsonl 2>&1
timeout 900 python tools/parareal_analysis.py fields --config c1 --variants classic --coarse-step 0.01 > gpurun_out/j_fields.jsonl 2>&1
timeout 900 python tools/parareal_analysis.py fields --config c1 --variants classic --coarse-step 0.004 >> gpurun_out/j_fields.jsonl 2>&1
timeout 900 python tools/parareal_analysis.py fields --config c1 --variants classic --mu-s 5e4 >> gpurun_out/j_fields.jsonl 2>&1
timeout 900 python tools/parareal_analysis.py fields --config c2 --iters 7 >> gpurun_out/j_fields.jsonl 2>&1
