# CGS passes A/B (Krylov counts + throughput), fused-Arnoldi re-check, GPU suite under PINT_CGS=1
for c in c2 c3 c4 c1; do
  for g in 1 2; do PINT_CGS=$g python bench.py --config $c --no-cpu-baseline > gpurun_out/cgs${g}_$c.json 2>/dev/null; done
done
for c in c1 c2; do PINT_FUSED=1 python bench.py --config $c --no-cpu-baseline > gpurun_out/fusedA_$c.json 2>/dev/null; done
PINT_CGS=1 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_cgs1.log 2>&1; tail -3 gpurun_out/t_cgs1.log
