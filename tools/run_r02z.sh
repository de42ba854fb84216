set -x
mkdir -p gpurun_out/r2z
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2z/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2z/gpu_tests.txt 2>&1
timeout 600 python tools/pipe_check.py > gpurun_out/r2z/pipe_check.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2z/bench_c2.json 2> gpurun_out/r2z/bench_c2.err
timeout 600 python bench.py --streams 56 --steps 3 --samples 4000 --no-cpu --no-e2e --kernel cluster > gpurun_out/r2z/bench_c2_s56.json 2> gpurun_out/r2z/bench_c2_s56.err
timeout 900 python bench.py --workload C5 --samples 2000 --as-shard-of 8 --steps 3 --no-cpu --no-e2e --kernel cluster > gpurun_out/r2z/bench_c5_g8_cluster.json 2> gpurun_out/r2z/bench_c5_g8_cluster.err
timeout 900 python bench.py --workload C5 --samples 2000 --as-shard-of 8 --steps 3 --no-cpu --no-e2e --kernel tc > gpurun_out/r2z/bench_c5_g8_tc.json 2> gpurun_out/r2z/bench_c5_g8_tc.err
