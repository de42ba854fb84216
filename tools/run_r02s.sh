set -x
mkdir -p gpurun_out/r2s
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2s/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "multi_stream_interleaved or one_cluster_per_stream or cluster_c3 or c2_full" > gpurun_out/r2s/pytest_pipe.log 2>&1
timeout 300 python tools/sweep_layers.py --layers 20,40 --n 8000 > gpurun_out/r2s/sweep_blocks.txt 2>&1
DVW_SKIP_RR=1 timeout 300 python tools/sweep_layers.py --layers 20,40 --n 8000 > gpurun_out/r2s/sweep_rr.txt 2>&1
for S in 16 32 56; do
  timeout 600 python bench.py --streams $S --steps 3 --samples 4000 --no-cpu --no-e2e --kernel cluster > gpurun_out/r2s/bench_c2_cl_s$S.json 2> gpurun_out/r2s/bench_c2_cl_s$S.err
done
DVW_SKIP_RR=1 timeout 600 python bench.py --streams 32 --steps 3 --samples 4000 --no-cpu --no-e2e --kernel cluster > gpurun_out/r2s/bench_c2_cl_s32_rr.json 2> gpurun_out/r2s/bench_c2_cl_s32_rr.err
timeout 900 python bench.py --workload C5 --samples 4000 --as-shard-of 8 --steps 3 --no-cpu --no-e2e --kernel cluster > gpurun_out/r2s/bench_c5_g8_cl.json 2> gpurun_out/r2s/bench_c5_g8_cl.err
