#!/bin/bash
# balanced warp roles of the staged residual alone vs the previous commit's build
mkdir -p gpurun_out
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/ai_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'e2e': d['e2e']['value'], 'solver': d['solver'], 'parity': d.get('parity'), 'clocks': d['clocks']}))" >> gpurun_out/ai_ab.jsonl
}
for rep in 1 2; do
run new c3 3 PINT_X=1
run prev c3 3 PINT_LIB=$PWD/scratch/libpint_prev.so
done
run new c4 5 PINT_X=1
run prev c4 5 PINT_LIB=$PWD/scratch/libpint_prev.so
run new c2 10 PINT_X=1
run prev c2 10 PINT_LIB=$PWD/scratch/libpint_prev.so
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q > gpurun_out/ai_tests.log 2>&1
true
