#!/bin/bash
# re-entry check (session 5): GPU suite, smoke, c3 bench + reference arm at the current commit
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/s_gpu_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/s_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s_smoke.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/s_bench_c3.json 2> gpurun_out/s_bench_c3.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s_bench_ref.json 2> gpurun_out/s_bench_ref.err
true
