#!/bin/bash
mkdir -p gpurun_out
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/aq_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'solver': d['solver']}))" >> gpurun_out/aq_ab.jsonl
}
for cfg_steps in "c2 10" "c1 10" "c4 5" "c3 3"; do
  set -- $cfg_steps
  run gate0_12 $1 $2 PINT_X=1
  run gate0_8 $1 $2 PINT_GATE0=8
  run gate0_6 $1 $2 PINT_GATE0=6
  run gate0_4 $1 $2 PINT_GATE0=4
  run gate0_6_gate2 $1 $2 PINT_GATE0=6 PINT_GATE=2
done
true
