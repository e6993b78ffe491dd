#!/bin/bash
# balanced warp roles of the staged residual + batched loads in the Givens / partial-sum tails: tests + A/B vs the previous commit's build
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_propagator.py tests/test_gpu_device_loop.py -m gpu -x -q > gpurun_out/ah_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/ah_tests.log
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/ah_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'e2e': d['e2e']['value'], 'solver': d['solver'], 'parity': d.get('parity'), 'clocks': d['clocks']}))" >> gpurun_out/ah_ab.jsonl
}
for cfg_steps in "c3 3" "c2 10" "c4 5" "c1 10"; do
  set -- $cfg_steps
  run new $1 $2 PINT_X=1
  run prev $1 $2 PINT_LIB=$PWD/scratch/libpint_prev.so
done
run new c3 3 PINT_X=1
run prev c3 3 PINT_LIB=$PWD/scratch/libpint_prev.so
true
