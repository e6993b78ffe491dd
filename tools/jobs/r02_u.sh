#!/bin/bash
# block-stencil Vanka sweep + staged fp32 residual: kernel tests, then A/B bench lines on c3 / c2 / c4
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q > gpurun_out/u_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/u_tests.log
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/u_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'e2e': d['e2e']['value'], 'solver': d['solver'], 'roofline': {k: d['roofline'][k] for k in ('kernel','frac','avg_launch_us','share_of_step')}, 'parity': d.get('parity'), 'clocks': d['clocks']}))" >> gpurun_out/u_ab.jsonl
}
run stencil+staged c3 3 PINT_X=1
run fused+staged   c3 3 PINT_VANKA=fused
run stencil+node   c3 3 PINT_SPMV32=node
run stencil+staged c2 10 PINT_X=1
run fused+staged   c2 10 PINT_VANKA=fused
run stencil+staged c4 5 PINT_X=1
run split+staged   c4 5 PINT_VANKA=split
run stencil+node   c4 5 PINT_SPMV32=node
run stencil+staged c1 10 PINT_X=1
run fused          c1 10 PINT_VANKA=fused
true
