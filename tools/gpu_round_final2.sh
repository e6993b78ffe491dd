# round-1 final measurements (second pass): smoke, GPU suite, bench lines c1-c4 (+CPU legs), reference arm,
# device Parareal c1, c2 launch list
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/y_smoke.log 2>&1; tail -1 gpurun_out/y_smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/y_tests.log 2>&1; tail -1 gpurun_out/y_tests.log
python bench.py > gpurun_out/y_bench_c2.json 2> gpurun_out/y_bench_c2.err
python bench.py --impl reference > gpurun_out/y_bench_ref.json 2> gpurun_out/y_bench_ref.err
for c in c1 c3 c4; do python bench.py --config $c > gpurun_out/y_bench_$c.json 2> gpurun_out/y_bench_$c.err; done
timeout 600 python tools/parareal_run.py --config c1 --driver device > gpurun_out/y_parareal_c1.json 2> gpurun_out/y_parareal_c1.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none \
    --nvtx --nvtx-include prof/ --csv --log-file gpurun_out/y_launches_c2.csv python tools/profile_step.py --config c2 --steps 8 > /dev/null 2>&1
