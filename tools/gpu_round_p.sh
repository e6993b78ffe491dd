timeout 900 python -m pytest tests -m gpu -q > gpurun_out/p_tests.log 2>&1; tail -1 gpurun_out/p_tests.log
for c in c2 c1 c3 c4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/p_$c.json 2>/dev/null; done
