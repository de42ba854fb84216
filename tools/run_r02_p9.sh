set -x
mkdir -p gpurun_out/p9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p9/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p9/gpu_tests.txt 2>&1
for G in 8 4 2 1; do
  timeout 1200 python bench.py --workload C5 --samples 8000 --as-shard-of $G --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/p9/bench_c5_g$G.json 2> gpurun_out/p9/bench_c5_g$G.err
done
for S in 8 16 32 56 112; do
  timeout 600 python bench.py --streams $S --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/p9/bench_c2_s$S.json 2> gpurun_out/p9/bench_c2_s$S.err
done
