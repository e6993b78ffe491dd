for c in c2 c1; do
  python bench.py --config $c --no-cpu-baseline > gpurun_out/k_def_$c.json 2>/dev/null
  for v in p2_8 p8_8; do PINT_LIB=scratch/lib_$v.so python bench.py --config $c --no-cpu-baseline > gpurun_out/k_${v}_$c.json 2>/dev/null; done
done
python bench.py --config c4 --no-cpu-baseline > gpurun_out/k_def_c4.json 2>/dev/null
for v in p4_4 p4_16; do PINT_LIB=scratch/lib_$v.so python bench.py --config c4 --no-cpu-baseline > gpurun_out/k_${v}_c4.json 2>/dev/null; done
