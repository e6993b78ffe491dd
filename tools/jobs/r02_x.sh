#!/bin/bash
# stencil-form Vanka inside the V-cycle tail + tail cluster rule: GPU suite, bench lines c1-c4, c1 device Parareal
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/x_gpu_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/x_gpu_tests.log
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/x_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'e2e': d['e2e']['value'], 'solver': d['solver'], 'roofline': {k: d['roofline'][k] for k in ('kernel','frac','avg_launch_us','share_of_step')}, 'clocks': d['clocks']}))" >> gpurun_out/x_ab.jsonl
}
run default c3 3 PINT_X=1
run default c2 10 PINT_X=1
run default c4 5 PINT_X=1
run default c1 10 PINT_X=1
run cell_inverses c1 10 PINT_VANKA=fused
run cell_inverses c2 10 PINT_VANKA=fused
run tail_cl4 c1 10 PINT_TAIL_CL=4
run tail_cl8 c1 10 PINT_TAIL_CL=8
for cl in 8 4 2; do
  PINT_TAIL_CL=$cl timeout 600 python tools/parareal_run.py --config c1 --driver device 2>> gpurun_out/x_par.err | sed "s/^/PINT_TAIL_CL=$cl /" >> gpurun_out/x_parareal_c1.log
done
true
