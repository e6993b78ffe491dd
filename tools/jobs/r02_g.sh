#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/g_gpu.log 2>&1
timeout 1800 python tools/c5_sweep.py --sizes 1e6 --slices 32 64 > gpurun_out/g_c5_lean.jsonl 2> gpurun_out/g_c5_lean.err
