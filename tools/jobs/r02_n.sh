#!/bin/bash
# node-owner strip Jacobian (k_jacobian_strip) + node-per-thread fp32 SpMV (k_spmv_node): tests, A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_configs.py -q -x > gpurun_out/n_tests.log 2>&1
timeout 900 python tools/elem_ab.py --cases c3 c2 c5_1e5x16 c5_1e6x8 --variants "" PINT_JAC=colour > gpurun_out/n_elem.jsonl 2> gpurun_out/n_elem.err
timeout 900 python tools/loop_ab.py --config c3 --steps 2 "PINT_X=0" PINT_JAC=colour PINT_SPMV32=row > gpurun_out/n_ab.jsonl 2> gpurun_out/n_ab.err
timeout 900 python tools/loop_ab.py --config c2 --steps 5 "PINT_X=0" PINT_JAC=colour PINT_SPMV32=row >> gpurun_out/n_ab.jsonl 2>> gpurun_out/n_ab.err
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/n_gpu.log 2>&1
true
