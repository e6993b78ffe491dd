#!/bin/bash
# inexact-Newton forcing: Krylov tolerance of the second Newton iteration (forcing * target) and of the first (rtol_first)
mkdir -p gpurun_out
run() {  # name config steps extra-args env...
  local name=$1 cfg=$2 steps=$3 extra=$4; shift 4
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline $extra 2>> gpurun_out/am_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'solver': d['solver'], 'parity': d.get('parity') and {k: d['parity'][k] for k in ('v','u','p','pass')}}))" >> gpurun_out/am_ab.jsonl
}
for cfg_steps in "c3 2" "c4 4" "c2 8"; do
  set -- $cfg_steps
  run forcing0.1 $1 $2 "" PINT_X=1
  run forcing0.25 $1 $2 "" PINT_FORCING=0.25
  run forcing0.5 $1 $2 "" PINT_FORCING=0.5
  run forcing1.0 $1 $2 "" PINT_FORCING=1.0
  run rtol_first1e-4 $1 $2 "--rtol-first 1e-4" PINT_X=1
  run rtol_first1e-5 $1 $2 "--rtol-first 1e-5" PINT_X=1
done
true
