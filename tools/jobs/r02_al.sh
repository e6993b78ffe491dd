#!/bin/bash
# closing check: full GPU suite, smoke, bench lines of every config + reference arm at the current commit
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/al_gpu_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/al_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/al_smoke.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/al_bench_ref.json 2> gpurun_out/al_bench_ref.err
timeout 900 python bench.py > gpurun_out/al_bench_c3.json 2> gpurun_out/al_bench_c3.err
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 > gpurun_out/al_bench_c2.json 2> gpurun_out/al_bench_c2.err
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/al_bench_c4.json 2> gpurun_out/al_bench_c4.err
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 > gpurun_out/al_bench_c1.json 2> gpurun_out/al_bench_c1.err
true
