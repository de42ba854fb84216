set -x
mkdir -p gpurun_out/r2t
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2t/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "multi_stream_interleaved or one_cluster_per_stream or cluster_c3 or c2_full or auto_routes" > gpurun_out/r2t/pytest_pipe.log 2>&1
timeout 300 python tools/sweep_layers.py --layers 20,40 --n 8000 > gpurun_out/r2t/sweep.txt 2>&1
for S in 16 32 56; do
  timeout 600 python bench.py --streams $S --steps 3 --samples 4000 --no-cpu --no-e2e --kernel cluster > gpurun_out/r2t/bench_c2_cl_s$S.json 2> gpurun_out/r2t/bench_c2_cl_s$S.err
done
timeout 900 python bench.py --workload C5 --samples 4000 --as-shard-of 8 --steps 3 --no-cpu --no-e2e --kernel cluster > gpurun_out/r2t/bench_c5_g8_cl.json 2> gpurun_out/r2t/bench_c5_g8_cl.err
timeout 900 python bench.py --workload C5 --samples 2000 --as-shard-of 4 --steps 3 --no-cpu --no-e2e --kernel cluster > gpurun_out/r2t/bench_c5_g4_cl.json 2> gpurun_out/r2t/bench_c5_g4_cl.err
