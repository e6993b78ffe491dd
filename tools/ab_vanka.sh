set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
for c in c2 c3 c4 c1; do
  python bench.py --config $c --no-cpu-baseline > gpurun_out/ab_fused_$c.json 2>/dev/null
  PINT_VANKA=split python bench.py --config $c --no-cpu-baseline > gpurun_out/ab_split_$c.json 2>/dev/null
  python -c "
import json
for k in ('fused','split'):
    d=json.load(open('gpurun_out/ab_%s_$c.json'%k)); r=d['roofline']
    print('$c',k,round(d['value'],1),d['config'].get('krylov_per_newton'),r['kernel'][:16],round(r['frac'],3),round(r['avg_launch_us'],2))
"
done
