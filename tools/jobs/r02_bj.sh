#!/bin/bash
# 3-d staged residual with moderate register caps (three builds) against the (node, row) kernel
mkdir -p gpurun_out
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/bj_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'solver': d['solver'], 'parity': d.get('parity') and d['parity']['pass']}))" >> gpurun_out/bj_ab.jsonl
}
run row_kernel c4 5 PINT_X=1
for v in 4 6 8; do
  run staged_minb$v c4 5 PINT_LIB=$PWD/scratch/libpint_rb$v.so PINT_SPMV32_MIN=50000
done
run row_kernel c4 5 PINT_X=1
true
