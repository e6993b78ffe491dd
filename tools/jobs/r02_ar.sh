#!/bin/bash
# whole Parareal runs with the final defaults (forcing target/2, reuse 64): device vs pipelined drivers
mkdir -p gpurun_out
timeout 300 python tools/parareal_run.py --config c1 --driver device >> gpurun_out/ar_parareal.jsonl 2>> gpurun_out/ar.err
timeout 300 python tools/parareal_run.py --config c1 --driver pipelined --chunks 2 >> gpurun_out/ar_parareal.jsonl 2>> gpurun_out/ar.err
timeout 600 python tools/parareal_run.py --config c2 --coarse-theta0 25 --driver device >> gpurun_out/ar_parareal.jsonl 2>> gpurun_out/ar.err
timeout 600 python tools/parareal_run.py --config c2 --coarse-theta0 25 --driver pipelined --chunks 4 >> gpurun_out/ar_parareal.jsonl 2>> gpurun_out/ar.err
timeout 900 python tools/parareal_run.py --config c3 --iters 3 --driver device >> gpurun_out/ar_parareal.jsonl 2>> gpurun_out/ar.err
timeout 900 python tools/parareal_run.py --config c3 --iters 3 --driver pipelined --chunks 4 >> gpurun_out/ar_parareal.jsonl 2>> gpurun_out/ar.err
timeout 900 python tools/parareal_run.py --config c4 --iters 3 --driver device >> gpurun_out/ar_parareal.jsonl 2>> gpurun_out/ar.err
timeout 900 python tools/parareal_run.py --config c3 --coarse-theta0 64 --iters 4 --driver device >> gpurun_out/ar_parareal.jsonl 2>> gpurun_out/ar.err
timeout 900 python tools/parareal_run.py --config c4 --coarse-theta0 25 --iters 4 --driver device >> gpurun_out/ar_parareal.jsonl 2>> gpurun_out/ar.err
true
