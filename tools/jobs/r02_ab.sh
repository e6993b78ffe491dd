#!/bin/bash
# V-cycle smoothing sweep on c3 / c4 with the stencil-form sweeps (Krylov count vs cost per iteration)
mkdir -p gpurun_out
for cfg in c3 c4; do
for a in "--pre 1 --post 1" "--pre 2 --post 2" "--pre 1 --post 2" "--pre 2 --post 1" "--omega 1.0" "--omega 0.8" "--omega 0.7"; do
  timeout 600 python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline $a 2>> gpurun_out/ab_sweep.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'args': '$a', 'config': '$cfg', 'value': d['value'], 'solver': d['solver']}))" >> gpurun_out/ab_sweep.jsonl
done
done
true
