#!/bin/bash
# omega = 1.0 as the 2-d default: GPU suite, whole Parareal runs, bench lines
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/bd_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/bd_tests.log
timeout 300 python tools/parareal_run.py --config c1 --driver device >> gpurun_out/bd_parareal.jsonl 2>> gpurun_out/bd.err
timeout 600 python tools/parareal_run.py --config c2 --coarse-theta0 25 --driver device >> gpurun_out/bd_parareal.jsonl 2>> gpurun_out/bd.err
timeout 900 python tools/parareal_run.py --config c3 --iters 3 --driver device >> gpurun_out/bd_parareal.jsonl 2>> gpurun_out/bd.err
timeout 900 python tools/parareal_run.py --config c3 --coarse-theta0 64 --iters 3 --driver pipelined --chunks 4 >> gpurun_out/bd_parareal.jsonl 2>> gpurun_out/bd.err
timeout 900 python bench.py > gpurun_out/bd_bench_c3.json 2> gpurun_out/bd_bench_c3.err
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 > gpurun_out/bd_bench_c2.json 2> gpurun_out/bd_bench_c2.err
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 > gpurun_out/bd_bench_c1.json 2> gpurun_out/bd_bench_c1.err
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/bd_bench_c4.json 2> gpurun_out/bd_bench_c4.err
true
