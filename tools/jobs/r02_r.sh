#!/bin/bash
# re-entry check: GPU suite, smoke, c3 and c2 bench lines at the current commit
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r_gpu_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r_smoke.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r_bench_c3.json 2> gpurun_out/r_bench_c3.err
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 > gpurun_out/r_bench_c2.json 2> gpurun_out/r_bench_c2.err
true
