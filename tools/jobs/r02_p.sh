#!/bin/bash
# full-step A/B: strip Jacobian v2 vs colour scatter (c3, c2, c1), GPU kernel tests
mkdir -p gpurun_out
timeout 900 python tools/loop_ab.py --config c3 --steps 2 "PINT_X=0" PINT_JAC=colour "PINT_X=0" PINT_JAC=colour > gpurun_out/p_ab.jsonl 2> gpurun_out/p_ab.err
timeout 900 python tools/loop_ab.py --config c2 --steps 5 "PINT_X=0" PINT_JAC=colour "PINT_X=0" PINT_JAC=colour >> gpurun_out/p_ab.jsonl 2>> gpurun_out/p_ab.err
timeout 900 python tools/loop_ab.py --config c1 --steps 5 "PINT_X=0" PINT_JAC=colour >> gpurun_out/p_ab.jsonl 2>> gpurun_out/p_ab.err
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/p_tests.log 2>&1
true
