#!/bin/bash
mkdir -p gpurun_out
run() {  # name config steps extra
  local name=$1 cfg=$2 steps=$3 extra=$4
  timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline $extra 2>> gpurun_out/ap_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'solver': d['solver'], 'parity': d.get('parity') and d['parity']['pass']}))" >> gpurun_out/ap_ab.jsonl
}
for cfg_steps in "c3 3" "c4 5" "c2 10" "c1 10"; do
  set -- $cfg_steps
  run reuse32 $1 $2 "--reuse 32"
  run reuse64 $1 $2 "--reuse 64"
  run reuse16 $1 $2 "--reuse 16"
done
true
