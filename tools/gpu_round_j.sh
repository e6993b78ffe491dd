timeout 900 python -m pytest tests -m gpu -q > gpurun_out/j_tests.log 2>&1; tail -1 gpurun_out/j_tests.log
for c in c2 c3 c4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/j_def_$c.json 2>/dev/null; done
PINT_VANKA=fused python bench.py --config c4 --no-cpu-baseline > gpurun_out/j_fused_c4.json 2>/dev/null
