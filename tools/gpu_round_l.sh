timeout 900 python -m pytest tests -m gpu -q > gpurun_out/l_tests.log 2>&1; tail -1 gpurun_out/l_tests.log
for c in c2 c3 c1 c4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/l_$c.json 2>/dev/null; done
