#!/bin/bash
# prolongation fused into the post-smoothing residual: kernel tests + A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q > gpurun_out/z_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/z_tests.log
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/z_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'e2e': d['e2e']['value'], 'solver': d['solver'], 'clocks': d['clocks']}))" >> gpurun_out/z_ab.jsonl
}
run fused_prolong c3 3 PINT_X=1
run separate_prolong c3 3 PINT_FUSE_PROLONG=0
run fused_prolong c4 5 PINT_X=1
run separate_prolong c4 5 PINT_FUSE_PROLONG=0
run fused_prolong c3 3 PINT_X=1
run separate_prolong c3 3 PINT_FUSE_PROLONG=0
true
