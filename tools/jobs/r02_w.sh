#!/bin/bash
# groups of slices on separate contexts / streams (overlap of the compute- and latency-bound phases); tail cluster size on c2
mkdir -p gpurun_out
timeout 1200 python tools/dual_stream_ab.py --config c3 --steps 16 --groups 1 2 4 > gpurun_out/w_dual_c3.jsonl 2> gpurun_out/w_dual_c3.err
timeout 600 python tools/dual_stream_ab.py --config c2 --steps 32 --groups 1 2 4 > gpurun_out/w_dual_c2.jsonl 2> gpurun_out/w_dual_c2.err
timeout 600 python tools/dual_stream_ab.py --config c4 --steps 16 --groups 1 2 4 > gpurun_out/w_dual_c4.jsonl 2> gpurun_out/w_dual_c4.err
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/w_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'e2e': d['e2e']['value'], 'solver': d['solver'], 'clocks': d['clocks']}))" >> gpurun_out/w_ab.jsonl
}
run tail_cl8 c2 10 PINT_TAIL_CL=8
run tail_cl4 c2 10 PINT_TAIL_CL=4
run tail_cl8 c4 5 PINT_TAIL_CL=8
run tail_cl4 c4 5 PINT_TAIL_CL=4
true
