#!/bin/bash
# re-entry check of HEAD: GPU suite, smoke, c3 / c2 bench lines
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/k_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/k_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/k_gpu.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/k_bench_c3.json 2> gpurun_out/k_bench_c3.err
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/k_bench_c2.json 2> gpurun_out/k_bench_c2.err
true
