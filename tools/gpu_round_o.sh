timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k "vanka" > gpurun_out/o_tests.log 2>&1; tail -1 gpurun_out/o_tests.log
for c in c2 c3; do
  python bench.py --config $c --no-cpu-baseline > gpurun_out/o_ch2_$c.json 2>/dev/null
  for v in ch1 ch4; do PINT_LIB=scratch/lib_$v.so python bench.py --config $c --no-cpu-baseline > gpurun_out/o_${v}_$c.json 2>/dev/null; done
done
