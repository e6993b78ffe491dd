#!/bin/bash
# register caps on the stencil sweep / staged residual; tiles rule; staged residual in 3-d again
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_propagator.py -m gpu -x -q > gpurun_out/bh_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/bh_tests.log
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/bh_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'roof': d['roofline']['frac'], 'us': d['roofline']['avg_launch_us'], 'solver': d['solver'], 'parity': d.get('parity') and d['parity']['pass']}))" >> gpurun_out/bh_ab.jsonl
}
for rep in 1 2; do
run wave_rule c4 5 PINT_X=1
run tiles1 c4 5 PINT_STENCIL_TILES=1
done
run staged3d_min50000 c4 5 PINT_SPMV32_MIN=50000
run staged3d_min0 c4 5 PINT_SPMV32_MIN=0
run wave_rule c3 3 PINT_X=1
run tiles1 c3 3 PINT_STENCIL_TILES=1
run wave_rule c3 3 PINT_X=1
run wave_rule c2 10 PINT_X=1
run tiles1 c2 10 PINT_STENCIL_TILES=1
run staged_min0 c2 10 PINT_SPMV32_MIN=0
true
