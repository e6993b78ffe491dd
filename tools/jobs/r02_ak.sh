#!/bin/bash
mkdir -p gpurun_out
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/ak_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'e2e': d['e2e']['value'], 'solver': d['solver'], 'clocks': d['clocks']}))" >> gpurun_out/ak_ab.jsonl
}
run default c4 5 PINT_X=1
run node_min0 c4 5 PINT_SPMV32=node PINT_SPMV32_MIN=0
run node_min50000 c4 5 PINT_SPMV32=node PINT_SPMV32_MIN=50000
run omega1 c2 10 PINT_X=1 
true
