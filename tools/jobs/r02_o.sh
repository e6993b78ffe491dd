#!/bin/bash
# strip Jacobian v2 (q-major phase-1 lanes): timing + ncu --set full of one strip launch and one colour launch on c3
mkdir -p gpurun_out
timeout 600 python tools/elem_ab.py --cases c3 c2 --variants "" PINT_JAC=colour > gpurun_out/o_elem.jsonl 2> gpurun_out/o_elem.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_jacobian_strip" -c 1 -o gpurun_out/o_strip \
  python tools/elem_ab.py --cases c3 --variants "" > gpurun_out/o_ncu.log 2>&1
ncu -i gpurun_out/o_strip.ncu-rep --page raw --csv > gpurun_out/o_strip_raw.csv 2>/dev/null
ncu -i gpurun_out/o_strip.ncu-rep --page source --csv > gpurun_out/o_strip_source.csv 2>/dev/null
rm -f gpurun_out/o_strip.ncu-rep
true
