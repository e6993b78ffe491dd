#!/bin/bash
mkdir -p gpurun_out
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/ao_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'solver': d['solver']}))" >> gpurun_out/ao_ab.jsonl
}
run default c2 10 PINT_X=1
run staged_fuseprolong c2 10 PINT_SPMV32_MIN=0 PINT_FUSE_PROLONG=1
run staged c2 10 PINT_SPMV32_MIN=0
run default c2 10 PINT_X=1
run reuse64 c3 3 PINT_X=1
true
