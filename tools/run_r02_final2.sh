mkdir -p gpurun_out/f2
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f2/smoke.log 2>&1
python bench.py > gpurun_out/f2/bench_c2.json 2> gpurun_out/f2/bench_c2.err
python bench.py --workload C3 --steps 3 --no-cpu > gpurun_out/f2/bench_c3.json 2> gpurun_out/f2/bench_c3.err
python bench.py --streams 56 --steps 3 --no-cpu > gpurun_out/f2/bench_c2_s56.json 2> gpurun_out/f2/bench_c2_s56.err
python bench.py --workload C5 --as-shard-of 8 --samples 8000 --steps 3 --no-cpu --no-e2e > gpurun_out/f2/bench_c5_g8.json 2> gpurun_out/f2/bench_c5_g8.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f2/bench_ref.json 2> gpurun_out/f2/bench_ref.err
