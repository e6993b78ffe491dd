#!/bin/bash
# V-cycle smoothing sweep on c3 / c2 (Krylov count vs cost per iteration)
mkdir -p gpurun_out
for a in "--pre 1 --post 1" "--pre 2 --post 2" "--pre 1 --post 2" "--pre 2 --post 1" "--omega 1.0" "--omega 0.8"; do
  timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline $a | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'args': '$a', 'config': 'c3', 'value': d['value'], 'solver': d['solver']}))" >> gpurun_out/q_sweep.jsonl 2>> gpurun_out/q_sweep.err
done
for a in "--pre 1 --post 1" "--pre 2 --post 2" "--pre 1 --post 2" "--omega 1.0"; do
  timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline $a | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'args': '$a', 'config': 'c2', 'value': d['value'], 'solver': d['solver']}))" >> gpurun_out/q_sweep.jsonl 2>> gpurun_out/q_sweep.err
done
true
