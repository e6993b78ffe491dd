#!/bin/bash
# round-2 closing profiles at the current commit: c3 launch list (time + DRAM bytes), ncu --set full of the
# sweep / residual / Krylov SpMV / Jacobian on c3 and of the 3-d sweep + residual on c4, c2 launch list
mkdir -p gpurun_out
export PINT_DEVICE_LOOP=0   # host-driven loop: the same kernels, launched one by one
timeout 600 python tools/profile_step.py --config c3 --steps 2 > gpurun_out/ag_plain_c3.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --nvtx --nvtx-include "prof/" --csv --log-file gpurun_out/ag_launches_c3.csv \
  python tools/profile_step.py --config c3 --steps 2 > gpurun_out/ag_ncu_launch_c3.log 2>&1
gzip -f gpurun_out/ag_launches_c3.csv
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --nvtx --nvtx-include "prof/" --csv --log-file gpurun_out/ag_launches_c4.csv \
  python tools/profile_step.py --config c4 --steps 2 > gpurun_out/ag_ncu_launch_c4.log 2>&1
gzip -f gpurun_out/ag_launches_c4.csv
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --nvtx --nvtx-include "prof/" --csv --log-file gpurun_out/ag_launches_c2.csv \
  python tools/profile_step.py --config c2 --steps 2 > gpurun_out/ag_ncu_launch_c2.log 2>&1
gzip -f gpurun_out/ag_launches_c2.csv
timeout 1800 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "prof/" \
  -k regex:"k_vanka_stencil_apply|k_resid32_staged|k_spmv|k_jacobian_strip|k_elem_tile|k_mdot_fused|k_mupdate_norm" -c 14 -o gpurun_out/ag_c3_full \
  python tools/profile_step.py --config c3 --steps 1 > gpurun_out/ag_ncu_c3.log 2>&1
ncu -i gpurun_out/ag_c3_full.ncu-rep --page raw --csv > gpurun_out/ag_c3_full_raw.csv 2>/dev/null
rm -f gpurun_out/ag_c3_full.ncu-rep
timeout 1800 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "prof/" \
  -k regex:"k_vanka_stencil_apply|k_resid32_staged|k_spmv" -c 8 -o gpurun_out/ag_c4_full \
  python tools/profile_step.py --config c4 --steps 1 > gpurun_out/ag_ncu_c4.log 2>&1
ncu -i gpurun_out/ag_c4_full.ncu-rep --page raw --csv > gpurun_out/ag_c4_full_raw.csv 2>/dev/null
rm -f gpurun_out/ag_c4_full.ncu-rep
true
