#!/bin/bash
# threshold of the staged residual kernel on the smaller configs
mkdir -p gpurun_out
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/aj_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'e2e': d['e2e']['value'], 'solver': d['solver'], 'clocks': d['clocks']}))" >> gpurun_out/aj_ab.jsonl
}
run default c4 5 PINT_X=1
run min0 c4 5 PINT_SPMV32_MIN=0
run min50000 c4 5 PINT_SPMV32_MIN=50000
run default c2 10 PINT_X=1
run min0 c2 10 PINT_SPMV32_MIN=0
run min30000 c2 10 PINT_SPMV32_MIN=30000
run default c3 3 PINT_X=1
run min0 c3 3 PINT_SPMV32_MIN=0
true
