timeout 900 python -m pytest tests -m gpu -q > gpurun_out/i_tests.log 2>&1; tail -1 gpurun_out/i_tests.log
for c in c2 c1 c3; do
  python bench.py --config $c --no-cpu-baseline > gpurun_out/i_hb1_$c.json 2>/dev/null
  PINT_HOST_BETA=0 python bench.py --config $c --no-cpu-baseline > gpurun_out/i_hb0_$c.json 2>/dev/null
done
