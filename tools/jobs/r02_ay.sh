#!/bin/bash
# multi-tangent strip Jacobian as the default: GPU suite, bench A/B, ncu --set full of the kernel
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/ay_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/ay_tests.log
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/ay_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'solver': d['solver'], 'parity': d.get('parity') and {k: d['parity'][k] for k in ('v','u','p','pass')}}))" >> gpurun_out/ay_ab.jsonl
}
for cfg_steps in "c3 3" "c2 10" "c1 10"; do
  set -- $cfg_steps
  run multi_tangent $1 $2 PINT_X=1
  run pass_per_direction $1 $2 PINT_JAC_MT=0
done
export PINT_DEVICE_LOOP=0
timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "prof/" \
  -k regex:"k_jacobian_strip" -c 2 -o gpurun_out/ay_jac_full \
  python tools/profile_step.py --config c3 --steps 1 > gpurun_out/ay_ncu.log 2>&1
ncu -i gpurun_out/ay_jac_full.ncu-rep --page raw --csv > gpurun_out/ay_jac_full_raw.csv 2>/dev/null
rm -f gpurun_out/ay_jac_full.ncu-rep
true
