set -x
mkdir -p gpurun_out/r2x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2x/build.log 2>&1
for M in 2 1 0; do
  DVW_PIPE_EARLY=$M timeout 600 python bench.py --streams 56 --steps 3 --samples 4000 --no-cpu --no-e2e --kernel cluster > gpurun_out/r2x/bench_c2_s56_m$M.json 2> gpurun_out/r2x/bench_c2_s56_m$M.err
  DVW_PIPE_EARLY=$M timeout 900 python bench.py --workload C5 --samples 2000 --as-shard-of 8 --steps 3 --no-cpu --no-e2e --kernel cluster > gpurun_out/r2x/bench_c5_g8_m$M.json 2> gpurun_out/r2x/bench_c5_g8_m$M.err
done
