set -x
mkdir -p gpurun_out/r2y
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2y/build.log 2>&1
timeout 600 python tools/pipe_check.py > gpurun_out/r2y/pipe_check.log 2>&1
timeout 600 python bench.py --streams 56 --steps 3 --samples 4000 --no-cpu --no-e2e --kernel cluster > gpurun_out/r2y/bench_c2_s56.json 2> gpurun_out/r2y/bench_c2_s56.err
timeout 900 python bench.py --workload C5 --samples 2000 --as-shard-of 8 --steps 3 --no-cpu --no-e2e --kernel cluster > gpurun_out/r2y/bench_c5_g8.json 2> gpurun_out/r2y/bench_c5_g8.err
