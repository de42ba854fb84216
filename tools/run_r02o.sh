set -x
mkdir -p gpurun_out/r2o
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2o/build.log 2>&1
for B in 1 0; do
  for G in 1 8 2 4; do
    DVW_BATCH_BALANCE=$B timeout 900 python bench.py --workload C5 --samples 8000 --as-shard-of $G --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2o/bench_c5_b${B}_g$G.json 2> gpurun_out/r2o/bench_c5_b${B}_g$G.err
  done
  DVW_BATCH_BALANCE=$B timeout 900 python bench.py --workload C4 --samples 20000 --no-cpu --no-e2e > gpurun_out/r2o/bench_c4_b$B.json 2> gpurun_out/r2o/bench_c4_b$B.err
done
DVW_BATCH_STAGES=2 timeout 900 python bench.py --workload C4 --samples 20000 --no-cpu --no-e2e > gpurun_out/r2o/bench_c4_st2.json 2> gpurun_out/r2o/bench_c4_st2.err
DVW_BATCH_STAGES=3 timeout 900 python bench.py --workload C4 --samples 20000 --no-cpu --no-e2e > gpurun_out/r2o/bench_c4_st3.json 2> gpurun_out/r2o/bench_c4_st3.err
