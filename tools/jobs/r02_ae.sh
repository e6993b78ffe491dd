#!/bin/bash
# round-2 c5 kernel roofline sweep with the stencil-form sweeps and the structural-zero products
mkdir -p gpurun_out
timeout 2400 python tools/c5_sweep.py --sizes 1e4 1e5 1e6 --slices 1 4 16 32 64 --mem-gb 120 > gpurun_out/ae_c5_sweep.jsonl 2> gpurun_out/ae_c5_sweep.err
true
