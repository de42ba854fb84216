set -x
mkdir -p gpurun_out/r2m
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2m/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "tc or batched or shard or sampler or quantized or auto or session" > gpurun_out/r2m/pytest_tc.log 2>&1
for G in 1 2 4 8; do
  timeout 900 python bench.py --workload C5 --samples 8000 --as-shard-of $G --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2m/bench_c5_g$G.json 2> gpurun_out/r2m/bench_c5_g$G.err
done
timeout 900 python bench.py --workload C4 --no-cpu > gpurun_out/r2m/bench_c4.json 2> gpurun_out/r2m/bench_c4.err
