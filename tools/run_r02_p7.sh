set -x
mkdir -p gpurun_out/p7
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p7/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p7/gpu_tests.txt 2>&1
timeout 600 python tools/pipe_check.py > gpurun_out/p7/pipe_check.log 2>&1
timeout 900 python bench.py --workload C3 --steps 3 --warmup 3 --samples 40000 --no-cpu --no-e2e > gpurun_out/p7/bench_c3.json 2> gpurun_out/p7/bench_c3.err
timeout 600 python tools/sweep_layers.py --layers 20,40 --n 8000 > gpurun_out/p7/sweep.txt 2>&1
timeout 600 python bench.py --workload C5 --samples 1000 --as-shard-of 8 --steps 3 --no-cpu --no-e2e --kernel cluster 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('C5x256 cluster', round(d['value']))" >> gpurun_out/p7/bench.txt
timeout 600 python bench.py --workload C5 --samples 1000 --as-shard-of 4 --steps 3 --no-cpu --no-e2e --kernel cluster 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('C5x512 cluster', round(d['value']))" >> gpurun_out/p7/bench.txt
