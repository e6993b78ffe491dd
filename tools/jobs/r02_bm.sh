#!/bin/bash
# staged V-cycle residual with fp32 accumulation (opt-in) vs fp64
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q > gpurun_out/bm_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/bm_tests.log
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/bm_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'solver': d['solver'], 'parity': d.get('parity') and {k: d['parity'][k] for k in ('v','u','p','pass')}}))" >> gpurun_out/bm_ab.jsonl
}
for rep in 1 2; do
run acc_f64 c3 3 PINT_X=1
run acc_f32 c3 3 PINT_RESID_ACC=f32
done
true
