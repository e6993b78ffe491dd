#!/bin/bash
# K1 in node-owner strips (one launch, no zeroing / colour scatter / fix-up): tests + A/B
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/as_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/as_tests.log
timeout 900 python tools/elem_ab.py --cases c3 c2 c5_1e5x16 --variants "" PINT_RES=tile > gpurun_out/as_elem.jsonl 2> gpurun_out/as_elem.err
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/as_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'solver': d['solver'], 'parity': d.get('parity') and {k: d['parity'][k] for k in ('v','u','p','pass')}}))" >> gpurun_out/as_ab.jsonl
}
for cfg_steps in "c3 3" "c2 10" "c1 10"; do
  set -- $cfg_steps
  run strip $1 $2 PINT_X=1
  run tile $1 $2 PINT_RES=tile
  run strip $1 $2 PINT_X=1
  run tile $1 $2 PINT_RES=tile
done
true
