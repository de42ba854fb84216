set -x
mkdir -p gpurun_out/r2v
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2v/build.log 2>&1
timeout 600 python tools/pipe_check.py > gpurun_out/r2v/pipe_check.log 2>&1
timeout 300 python tools/sweep_layers.py --layers 20,40 --n 8000 > gpurun_out/r2v/sweep.txt 2>&1
timeout 900 python bench.py --workload C5 --samples 4000 --as-shard-of 8 --steps 3 --no-cpu --no-e2e --kernel cluster > gpurun_out/r2v/bench_c5_g8_cl.json 2> gpurun_out/r2v/bench_c5_g8_cl.err
timeout 600 python bench.py --streams 56 --steps 3 --samples 4000 --no-cpu --no-e2e --kernel cluster > gpurun_out/r2v/bench_c2_cl_s56.json 2> gpurun_out/r2v/bench_c2_cl_s56.err
