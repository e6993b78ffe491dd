#!/bin/bash
# round 2, first device-loop check: GPU tests of the new paths, then c2/c3 bench (device loop vs host loop)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_device_loop.py -x -q > gpurun_out/a_loop.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_device_loop.py > gpurun_out/a_gpu.log 2>&1
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/a_bench_c2.json 2> gpurun_out/a_bench_c2.err
PINT_DEVICE_LOOP=0 timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/a_bench_c2_host.json 2> gpurun_out/a_bench_c2_host.err
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/a_bench_c1.json 2> gpurun_out/a_bench_c1.err
timeout 900 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/a_bench_c3.json 2> gpurun_out/a_bench_c3.err
timeout 900 python tools/parareal_run.py --config c1 > gpurun_out/a_parareal_c1.log 2>&1
timeout 900 python tools/parareal_run.py --config c1 --driver pipelined >> gpurun_out/a_parareal_c1.log 2>&1
timeout 900 python tools/parareal_run.py --config c2 >> gpurun_out/a_parareal_c1.log 2>&1
true
