#!/bin/bash
# structural-zero planes skipped by the product kernels: kernel tests, bitwise A/B against a -DPINT_PATTERN=0 build, bench A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q > gpurun_out/aa_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/aa_tests.log
timeout 600 python tools/pattern_ab.py gpurun_out/aa_pat.npz > gpurun_out/aa_pattern.log 2>&1
PINT_LIB=$PWD/scratch/libpint_nopat.so timeout 600 python tools/pattern_ab.py gpurun_out/aa_nopat.npz >> gpurun_out/aa_pattern.log 2>&1
python tools/pattern_ab.py --compare gpurun_out/aa_pat.npz gpurun_out/aa_nopat.npz >> gpurun_out/aa_pattern.log 2>&1
rm -f gpurun_out/aa_pat.npz gpurun_out/aa_nopat.npz
run() {  # name config steps env...
  local name=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>> gpurun_out/aa_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case': '$name', 'config': '$cfg', 'value': d['value'], 'e2e': d['e2e']['value'], 'solver': d['solver'], 'parity': d.get('parity'), 'clocks': d['clocks']}))" >> gpurun_out/aa_ab.jsonl
}
run skip_zero_planes c3 3 PINT_X=1
run full_loops c3 3 PINT_LIB=$PWD/scratch/libpint_nopat.so
run skip_zero_planes c4 5 PINT_X=1
run full_loops c4 5 PINT_LIB=$PWD/scratch/libpint_nopat.so
run skip_zero_planes c2 10 PINT_X=1
run full_loops c2 10 PINT_LIB=$PWD/scratch/libpint_nopat.so
run skip_zero_planes c1 10 PINT_X=1
run full_loops c1 10 PINT_LIB=$PWD/scratch/libpint_nopat.so
timeout 1200 python tools/dual_stream_ab.py --config c3 --steps 16 --groups 1 2 > gpurun_out/aa_dual_c3.jsonl 2> gpurun_out/aa_dual_c3.err
timeout 600 python tools/dual_stream_ab.py --config c4 --steps 16 --groups 1 2 > gpurun_out/aa_dual_c4.jsonl 2> gpurun_out/aa_dual_c4.err
true
