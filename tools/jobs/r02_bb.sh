#!/bin/bash
mkdir -p gpurun_out
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/bb_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'solver': d['solver'], 'parity': d.get('parity') and d['parity']['pass']}))" >> gpurun_out/bb_ab.jsonl
}
run tail2048 c4 5 PINT_X=1
run tail4000 c4 5 PINT_TAIL_ROWS=4000
run tail4000_cl8 c4 5 PINT_TAIL_ROWS=4000 PINT_TAIL_CL=8
run tail2048 c4 5 PINT_X=1
true
