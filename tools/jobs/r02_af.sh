#!/bin/bash
# tail: coarsest inverse staged in shared memory vs read from L2 (one wave of co-resident CTAs)
mkdir -p gpurun_out
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/af_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'e2e': d['e2e']['value'], 'solver': d['solver'], 'clocks': d['clocks']}))" >> gpurun_out/af_ab.jsonl
}
run rule c3 3 PINT_X=1
run stage1 c3 3 PINT_TAIL_STAGE=1
run stage0 c3 3 PINT_TAIL_STAGE=0
run rule c2 10 PINT_X=1
run stage0 c2 10 PINT_TAIL_STAGE=0
run rule c4 5 PINT_X=1
run stage0 c4 5 PINT_TAIL_STAGE=0
run rule c1 10 PINT_X=1
run stage0 c1 10 PINT_TAIL_STAGE=0
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_propagator.py -m gpu -x -q > gpurun_out/af_tests.log 2>&1
true
