#!/bin/bash
mkdir -p gpurun_out
PINT_FORCING=0.5 timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/an_tests_f05.log 2>&1
echo "pytest exit $?" >> gpurun_out/an_tests_f05.log
PINT_FORCING=0.25 timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/an_tests_f025.log 2>&1
echo "pytest exit $?" >> gpurun_out/an_tests_f025.log
for f in 0.1 0.5; do PINT_FORCING=$f timeout 300 python tools/parareal_run.py --config c1 --driver device | sed "s/^/PINT_FORCING=$f /" >> gpurun_out/an_par.log 2>&1; done
for f in 0.1 0.5; do PINT_FORCING=$f timeout 600 python tools/parareal_run.py --config c2 --coarse-theta0 25 --driver device | sed "s/^/PINT_FORCING=$f /" >> gpurun_out/an_par.log 2>&1; done
true
