#!/bin/bash
# lanes per row of the tail's stencil-form Vanka sweep (three builds), c3 bench with the parity fixture + reference arm
mkdir -p gpurun_out
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/y_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'e2e': d['e2e']['value'], 'solver': d['solver'], 'roofline': {k: d['roofline'][k] for k in ('kernel','frac','avg_launch_us','share_of_step')}, 'clocks': d['clocks']}))" >> gpurun_out/y_ab.jsonl
}
for cfg in c1 c2; do
  run pv1 $cfg 10 PINT_X=1
  run pv2 $cfg 10 PINT_LIB=$PWD/scratch/libpint_pv2.so
  run pv4 $cfg 10 PINT_LIB=$PWD/scratch/libpint_pv4.so
  run cell $cfg 10 PINT_VANKA=fused
done
run pv1 c4 5 PINT_X=1
run pv3_8 c4 5 PINT_LIB=$PWD/scratch/libpint_pv4.so
run cell c4 5 PINT_VANKA=split
run pv1 c3 3 PINT_X=1
run pv2 c3 3 PINT_LIB=$PWD/scratch/libpint_pv2.so
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/y_bench_c3.json 2> gpurun_out/y_bench_c3.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/y_bench_ref.json 2> gpurun_out/y_bench_ref.err
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -x -q > gpurun_out/y_cfg_tests.log 2>&1
true
