# ncu --set full of the c2 V-cycle tail and of the c4 fp32 residual SpMV (source-level stalls)
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include prof/ -k regex:k_vcycle_tail_cl -c 2 \
  -o gpurun_out/ncu_tail_c2 python tools/profile_step.py --config c2 --steps 1 > gpurun_out/ncu_tail.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include prof/ -k 'regex:k_spmv<3, 1, 3, float>|k_spmv' -c 3 \
  -o gpurun_out/ncu_spmv_c4 python tools/profile_step.py --config c4 --steps 1 > gpurun_out/ncu_spmv.log 2>&1
ls -la gpurun_out/*.ncu-rep
