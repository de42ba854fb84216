mkdir -p gpurun_out/p22
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "multi_stream or auto_routes" > gpurun_out/p22/tests_ms.txt 2>&1
timeout 600 python tools/pipe_check.py > gpurun_out/p22/pipe_check.log 2>&1
for r in 1 2; do
timeout 600 python bench.py --streams 56 --steps 3 --warmup 3 --samples 4000 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('C2 streams 56', round(d['value']))" >> gpurun_out/p22/bench.txt
timeout 600 python bench.py --workload C5 --samples 1000 --as-shard-of 8 --steps 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('C5x256', round(d['value']))" >> gpurun_out/p22/bench.txt
done
timeout 600 python tools/sweep_layers.py --layers 20,40 --n 8000 >> gpurun_out/p22/bench.txt 2>&1
