set -x
mkdir -p gpurun_out/r2l
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2l/build.log 2>&1
for G in 1 2 4 8; do
  timeout 900 python bench.py --workload C5 --samples 8000 --as-shard-of $G --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2l/bench_c5_g$G.json 2> gpurun_out/r2l/bench_c5_g$G.err
done
timeout 900 python bench.py --workload C1 > gpurun_out/r2l/bench_c1.json 2> gpurun_out/r2l/bench_c1.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_batch -c 1 -o gpurun_out/r2l/batch_c4 python tools/ncu_c4.py > gpurun_out/r2l/ncu_c4.log 2>&1
timeout 300 python tools/trace_batch.py > gpurun_out/r2l/trace_c4.log 2>&1
timeout 2400 python bench.py --workload C5 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2l/bench_c5_full.json 2> gpurun_out/r2l/bench_c5_full.err
