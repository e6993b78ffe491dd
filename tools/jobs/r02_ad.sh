#!/bin/bash
# device vs pipelined Parareal drivers (fine phase of iteration i+1 overlapping the sweep of iteration i)
mkdir -p gpurun_out
for rep in 1 2; do
timeout 300 python tools/parareal_run.py --config c1 --driver device >> gpurun_out/ad_parareal.jsonl 2>> gpurun_out/ad.err
timeout 300 python tools/parareal_run.py --config c1 --driver pipelined --chunks 2 >> gpurun_out/ad_parareal.jsonl 2>> gpurun_out/ad.err
timeout 300 python tools/parareal_run.py --config c1 --driver pipelined --chunks 5 >> gpurun_out/ad_parareal.jsonl 2>> gpurun_out/ad.err
done
timeout 600 python tools/parareal_run.py --config c2 --coarse-theta0 25 --driver device >> gpurun_out/ad_parareal.jsonl 2>> gpurun_out/ad.err
timeout 600 python tools/parareal_run.py --config c2 --coarse-theta0 25 --driver pipelined --chunks 4 >> gpurun_out/ad_parareal.jsonl 2>> gpurun_out/ad.err
timeout 600 python tools/parareal_run.py --config c2 --coarse-theta0 25 --driver pipelined --chunks 8 >> gpurun_out/ad_parareal.jsonl 2>> gpurun_out/ad.err
timeout 900 python tools/parareal_run.py --config c3 --iters 3 --driver device >> gpurun_out/ad_parareal.jsonl 2>> gpurun_out/ad.err
timeout 900 python tools/parareal_run.py --config c3 --iters 3 --driver pipelined --chunks 4 >> gpurun_out/ad_parareal.jsonl 2>> gpurun_out/ad.err
timeout 900 python tools/parareal_run.py --config c3 --iters 3 --driver pipelined --chunks 8 >> gpurun_out/ad_parareal.jsonl 2>> gpurun_out/ad.err
timeout 900 python tools/parareal_run.py --config c4 --iters 3 --driver device >> gpurun_out/ad_parareal.jsonl 2>> gpurun_out/ad.err
timeout 900 python tools/parareal_run.py --config c4 --iters 3 --driver pipelined --chunks 4 >> gpurun_out/ad_parareal.jsonl 2>> gpurun_out/ad.err
true
