timeout 900 python -m pytest tests -m gpu -q > gpurun_out/q_tests.log 2>&1; tail -1 gpurun_out/q_tests.log
for c in c2 c3 c1; do
  python bench.py --config $c --no-cpu-baseline > gpurun_out/q_def_$c.json 2>/dev/null
  PINT_DEFER_SCALE=0 python bench.py --config $c --no-cpu-baseline > gpurun_out/q_off_$c.json 2>/dev/null
done
