# round-1 final measurements: smoke, GPU suite, bench lines c1-c4 (+CPU legs), reference arm, device Parareal c1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.log 2>&1; tail -1 gpurun_out/z_smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/z_tests.log 2>&1; tail -1 gpurun_out/z_tests.log
python bench.py > gpurun_out/z_bench_c2.json 2> gpurun_out/z_bench_c2.err
python bench.py --impl reference > gpurun_out/z_bench_ref.json 2> gpurun_out/z_bench_ref.err
for c in c1 c3 c4; do python bench.py --config $c > gpurun_out/z_bench_$c.json 2> gpurun_out/z_bench_$c.err; done
timeout 600 python tools/parareal_run.py --config c1 --driver device > gpurun_out/z_parareal_c1.json 2> gpurun_out/z_parareal_c1.err
