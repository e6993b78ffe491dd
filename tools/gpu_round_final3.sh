# round-1 closing measurements at the final commit: smoke, bench lines c1-c4 (+CPU legs), reference arm
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/x_smoke.log 2>&1; tail -1 gpurun_out/x_smoke.log
python bench.py > gpurun_out/x_bench_c2.json 2> gpurun_out/x_bench_c2.err
python bench.py --impl reference > gpurun_out/x_bench_ref.json 2> gpurun_out/x_bench_ref.err
for c in c1 c3 c4; do python bench.py --config $c > gpurun_out/x_bench_$c.json 2> gpurun_out/x_bench_$c.err; done
