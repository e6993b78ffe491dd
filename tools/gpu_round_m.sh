for c in c2 c1; do
  PINT_SCALE_FUSE=16384 python bench.py --config $c --no-cpu-baseline > gpurun_out/m_sf_$c.json 2>/dev/null
  python bench.py --config $c --no-cpu-baseline > gpurun_out/m_def_$c.json 2>/dev/null
done
