mkdir -p gpurun_out/f3
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for G in 8 4 2 1; do
  timeout 1200 python bench.py --workload C5 --samples 8000 --as-shard-of $G --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/f3/bench_c5_g$G.json 2> gpurun_out/f3/bench_c5_g$G.err
done
timeout 900 python bench.py --workload C4 --steps 2 --warmup 3 --no-cpu --no-e2e --precision tf32 > gpurun_out/f3/bench_c4_tf32.json 2> gpurun_out/f3/bench_c4_tf32.err
