mkdir -p gpurun_out/f4
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f4/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f4/gpu_tests.txt 2>&1
timeout 1200 python bench.py --workload C5 --samples 8000 --as-shard-of 8 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/f4/bench_c5_g8.json 2> gpurun_out/f4/bench_c5_g8.err
timeout 1200 python bench.py --workload C5 --as-shard-of 8 --steps 3 --warmup 3 --cpu-samples 1600 --no-e2e > gpurun_out/f4/bench_c5_g8_full.json 2> gpurun_out/f4/bench_c5_g8_full.err
timeout 600 python bench.py --workload C5 --samples 1000 --as-shard-of 4 --steps 3 --no-cpu --no-e2e --kernel cluster 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('C5x512 cluster', round(d['value']))" > gpurun_out/f4/c5x512_cluster.txt
python bench.py > gpurun_out/f4/bench_c2.json 2> gpurun_out/f4/bench_c2.err
