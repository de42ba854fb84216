set -x
mkdir -p gpurun_out/r2r
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2r/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "multi_stream_interleaved" > gpurun_out/r2r/pytest_pipe.log 2>&1
timeout 300 python tools/sweep_layers.py --layers 20,40 --n 8000 > gpurun_out/r2r/sweep.txt 2>&1
for S in 8 16 32 64; do
  timeout 600 python bench.py --streams $S --steps 3 --samples 4000 --no-cpu --no-e2e --kernel cluster > gpurun_out/r2r/bench_c2_cl_s$S.json 2> gpurun_out/r2r/bench_c2_cl_s$S.err
done
timeout 900 python bench.py --workload C5 --samples 4000 --as-shard-of 8 --steps 3 --no-cpu --no-e2e --kernel cluster > gpurun_out/r2r/bench_c5_g8_cl.json 2> gpurun_out/r2r/bench_c5_g8_cl.err
timeout 900 python bench.py --workload C5 --samples 2000 --as-shard-of 1 --steps 2 --no-cpu --no-e2e --kernel cluster > gpurun_out/r2r/bench_c5_g1_cl.json 2> gpurun_out/r2r/bench_c5_g1_cl.err
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2r/pytest_all.log 2>&1
