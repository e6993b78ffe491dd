#!/bin/bash
# round-2 profiles: c3 launch list (time + DRAM bytes, 2 fine steps), ncu --set full of the
# element kernels + level-0 Vanka sweep on c3, and of k_vanka_cell / element kernels on c4
mkdir -p gpurun_out
export PINT_DEVICE_LOOP=0   # host-driven loop: the same kernels, launched one by one
timeout 600 python tools/profile_step.py --config c3 --steps 2 > gpurun_out/l_plain_c3.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --nvtx --nvtx-include "prof/" --csv --log-file gpurun_out/l_launches_c3.csv \
  python tools/profile_step.py --config c3 --steps 2 > gpurun_out/l_ncu_launch.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "prof/" \
  -k regex:"k_jacobian_lin|k_elem_tile|k_vanka_apply" -c 12 -o gpurun_out/l_c3_full \
  python tools/profile_step.py --config c3 --steps 1 > gpurun_out/l_ncu_c3.log 2>&1
timeout 600 python tools/profile_step.py --config c4 --steps 1 > gpurun_out/l_plain_c4.log 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "prof/" \
  -k regex:"k_jacobian_lin|k_elem_tile|k_vanka_cell" -c 12 -o gpurun_out/l_c4_full \
  python tools/profile_step.py --config c4 --steps 1 > gpurun_out/l_ncu_c4.log 2>&1
ls -la gpurun_out
true
# export on the box (the .ncu-rep files exceed gpurun's 64 MiB copy-back)
for r in l_c3_full l_c4_full; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page source --csv -k regex:"k_jacobian_lin|k_elem_tile" -c 3 > gpurun_out/${r}_source.csv 2>/dev/null
  rm -f gpurun_out/$r.ncu-rep
done
ls -la gpurun_out
