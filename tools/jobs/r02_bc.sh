#!/bin/bash
mkdir -p gpurun_out
for cfg_steps in "c3 3" "c2 10" "c1 10"; do
  set -- $cfg_steps
  for om in 0.9 1.0 0.95; do
  timeout 900 python bench.py --config $1 --steps $2 --warmup 3 --no-cpu-baseline --omega $om 2>> gpurun_out/bc.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'omega': $om, 'config': '$1', 'value': d['value'], 'solver': d['solver']}))" >> gpurun_out/bc_ab.jsonl
  done
done
true
