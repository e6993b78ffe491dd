# A/B of the fused CGS-norm kernel + ncu captures of the fused Vanka sweep
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "fused" > gpurun_out/t_fused.log 2>&1; tail -2 gpurun_out/t_fused.log
for c in c2 c3 c4; do
  python bench.py --config $c --no-cpu-baseline > gpurun_out/n_fused_$c.json 2>/dev/null
  PINT_SPLIT_NORM=1 python bench.py --config $c --no-cpu-baseline > gpurun_out/n_split_$c.json 2>/dev/null
done
for c in c2 c3; do
  cnt=4; [ $c = c3 ] && cnt=1
  timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include prof/ -k regex:k_vanka_apply -c $cnt \
    -o gpurun_out/ncu_vanka_apply_$c python tools/profile_step.py --config $c --steps 1 > gpurun_out/ncu_$c.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none \
  --nvtx --nvtx-include prof/ --csv --log-file gpurun_out/launches_c2.csv python tools/profile_step.py --config c2 --steps 8 > gpurun_out/ncu_l2.log 2>&1
ls gpurun_out
