# round-1 refresh: GPU suite, smoke, bench lines (c2 default + reference arm, c1/c3/c4), launch lists
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f_tests.log 2>&1; tail -2 gpurun_out/f_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; tail -1 gpurun_out/f_smoke.log
python bench.py > gpurun_out/f_bench_c2.json 2> gpurun_out/f_bench_c2.err
python bench.py --impl reference > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err
for c in c1 c3 c4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/f_bench_$c.json 2>/dev/null; done
for c in c2 c3 c4; do
  st=8; [ $c = c3 ] && st=2; [ $c = c4 ] && st=2
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none \
    --nvtx --nvtx-include prof/ --csv --log-file gpurun_out/f_launches_$c.csv python tools/profile_step.py --config $c --steps $st > /dev/null 2>&1
done
ls gpurun_out | grep "^f_"
