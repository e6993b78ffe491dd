python bench.py --config c4 --no-cpu-baseline > gpurun_out/h_occ4.json 2>/dev/null
PINT_LIB=scratch/lib_occ2.so python bench.py --config c4 --no-cpu-baseline > gpurun_out/h_occ2.json 2>/dev/null
PINT_LIB=scratch/lib_occ3.so python bench.py --config c4 --no-cpu-baseline > gpurun_out/h_occ3.json 2>/dev/null
python bench.py --config c4 --no-cpu-baseline > gpurun_out/h_occ4b.json 2>/dev/null
