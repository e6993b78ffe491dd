#!/bin/bash
# ncu --set full of the element kernels and the fp32 V-cycle SpMV on c3 (host loop: same kernels)
mkdir -p gpurun_out
export PINT_DEVICE_LOOP=0
timeout 600 python tools/profile_step.py --config c3 --steps 1 > gpurun_out/f_plain.log 2>&1 && \
timeout 2400 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "prof/" \
  -k regex:"k_jacobian_lin|k_residual_colour|k_spmv" -c 12 -o gpurun_out/f_c3_elem python tools/profile_step.py --config c3 --steps 1 > gpurun_out/f_ncu.log 2>&1
true
