#!/bin/bash
# Jacobian strip width (phase-2 rounds) and tail threshold with the stencil-form tail
mkdir -p gpurun_out
timeout 900 python tools/elem_ab.py --cases c3 c2 c5_1e5x16 --variants "" PINT_STRIP_W=31 PINT_STRIP_W=20 PINT_STRIP_W=16 > gpurun_out/ac_elem.jsonl 2> gpurun_out/ac_elem.err
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/ac_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'e2e': d['e2e']['value'], 'solver': d['solver'], 'clocks': d['clocks']}))" >> gpurun_out/ac_ab.jsonl
}
run tail2048 c3 3 PINT_X=1
run tail6000 c3 3 PINT_TAIL_ROWS=6000
run tail2048 c2 10 PINT_X=1
run tail6000 c2 10 PINT_TAIL_ROWS=6000
run tail2048 c4 5 PINT_X=1
run tail3000 c4 5 PINT_TAIL_ROWS=3000
run strip31 c3 3 PINT_STRIP_W=31
true
