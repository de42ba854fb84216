mkdir -p gpurun_out/p16
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "multi_stream or auto_routes" > gpurun_out/p16/tests_ms.txt 2>&1
timeout 600 python tools/pipe_check.py > gpurun_out/p16/pipe_check.log 2>&1
for a in "56 400" "14 400" "56 2000" "28 400" "9 300"; do timeout 120 python tools/pipe_smoke.py $a >> gpurun_out/p16/ptcheck.txt 2>&1; done
for X in 7 3; do
DVW_XPB=$X timeout 600 python bench.py --streams 56 --steps 3 --warmup 3 --samples 4000 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('xpb $X C2 streams 56', round(d['value']))" >> gpurun_out/p16/bench.txt
DVW_XPB=$X timeout 600 python bench.py --workload C5 --samples 1000 --as-shard-of 8 --steps 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('xpb $X C5x256', round(d['value']))" >> gpurun_out/p16/bench.txt
done
