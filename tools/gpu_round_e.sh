timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_e.log 2>&1; tail -2 gpurun_out/t_e.log
for c in c2 c1; do
  python bench.py --config $c --no-cpu-baseline > gpurun_out/e_fuse_$c.json 2>/dev/null
  PINT_SCALE_FUSE=0 python bench.py --config $c --no-cpu-baseline > gpurun_out/e_nofuse_$c.json 2>/dev/null
done
