#!/bin/bash
# compute-sanitizer memcheck on the small-problem GPU tests (host loop and device loop)
mkdir -p gpurun_out
SEL="tests/test_gpu_device_loop.py::test_device_loop_bitwise_equals_host_loop tests/test_gpu_device_loop.py::test_coarse_sweep_equals_per_slice_composition tests/test_gpu_kernels.py tests/test_gpu_propagator.py::test_window_matches_oracle"
timeout 600 python -m pytest -q -x $SEL > gpurun_out/san_plain.log 2>&1 && \
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report analysis --error-exitcode 9 --log-file gpurun_out/san_racecheck.txt \
  python -m pytest -q -x $SEL > gpurun_out/san_racecheck_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/san_racecheck_pytest.log
