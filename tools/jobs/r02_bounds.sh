#!/bin/bash
# GPU tests on a -DPINT_BOUNDS=1 build (device-side index checks in the round-2 kernels; the pool's
# compute-sanitizer is closed): kernel, config, propagator, device-loop and Parareal tests, the strip residual
# variant, and a 2-step c3 / c4 bench.  A violated check traps and fails the test with a CUDA error.
mkdir -p gpurun_out
export PINT_LIB=$PWD/scratch/libpint_bounds.so
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/bounds_tests.log 2>&1
echo "pytest exit $? (PINT_LIB=$PINT_LIB)" >> gpurun_out/bounds_tests.log
PINT_RES=strip timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_propagator.py -m gpu -q > gpurun_out/bounds_tests_resstrip.log 2>&1
echo "pytest exit $? (PINT_RES=strip)" >> gpurun_out/bounds_tests_resstrip.log
PINT_FUSE_PROLONG=1 PINT_SPMV32_MIN=0 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_propagator.py -m gpu -q > gpurun_out/bounds_tests_fuse.log 2>&1
echo "pytest exit $? (PINT_FUSE_PROLONG=1 PINT_SPMV32_MIN=0)" >> gpurun_out/bounds_tests_fuse.log
for cfg in c3 c4 c2; do
  timeout 900 python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline 2> gpurun_out/bounds_bench_$cfg.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'config': '$cfg', 'value_checked_build': d['value'], 'solver': d['solver'], 'parity': d['parity']}))" >> gpurun_out/bounds_bench.jsonl
done
grep -l "PINT_BOUNDS violated" gpurun_out/bounds_*.log gpurun_out/bounds_*.err > gpurun_out/bounds_violations.txt 2>/dev/null
echo "files with violations: $(wc -l < gpurun_out/bounds_violations.txt)" >> gpurun_out/bounds_tests.log
true
