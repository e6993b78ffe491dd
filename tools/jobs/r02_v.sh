#!/bin/bash
# after the block-stencil sweep: kernel tests, tail cluster size on c3, fresh c3 launch list, ncu --set full of the new kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q > gpurun_out/v_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/v_tests.log
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/v_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'e2e': d['e2e']['value'], 'solver': d['solver'], 'clocks': d['clocks']}))" >> gpurun_out/v_ab.jsonl
}
run tail_cl4 c3 3 PINT_TAIL_CL=4
run tail_cl8 c3 3 PINT_TAIL_CL=8
run tail_cl2 c3 3 PINT_TAIL_CL=2
export PINT_DEVICE_LOOP=0   # host-driven loop: the same kernels, launched one by one
timeout 600 python tools/profile_step.py --config c3 --steps 2 > gpurun_out/v_plain_c3.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --nvtx --nvtx-include "prof/" --csv --log-file gpurun_out/v_launches_c3.csv \
  python tools/profile_step.py --config c3 --steps 2 > gpurun_out/v_ncu_launch.log 2>&1
gzip -f gpurun_out/v_launches_c3.csv
timeout 1800 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "prof/" \
  -k regex:"k_vanka_stencil_apply|k_resid32_staged" -c 8 -o gpurun_out/v_c3_full \
  python tools/profile_step.py --config c3 --steps 1 > gpurun_out/v_ncu_c3.log 2>&1
ncu -i gpurun_out/v_c3_full.ncu-rep --page raw --csv > gpurun_out/v_c3_full_raw.csv 2>/dev/null
ncu -i gpurun_out/v_c3_full.ncu-rep --page details --csv > gpurun_out/v_c3_full_details.csv 2>/dev/null
rm -f gpurun_out/v_c3_full.ncu-rep
true
