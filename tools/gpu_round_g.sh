timeout 900 python -m pytest tests -m gpu -q > gpurun_out/g_tests.log 2>&1; tail -3 gpurun_out/g_tests.log
for c in c2 c3; do python bench.py --config $c --no-cpu-baseline > gpurun_out/g_bench_$c.json 2>/dev/null; done
