set -x
mkdir -p gpurun_out/p10
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p10/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "multi_stream or auto_routes" > gpurun_out/p10/tests_ms.txt 2>&1
timeout 600 python tools/pipe_check.py > gpurun_out/p10/pipe_check.log 2>&1
for S in 56 112 16; do
  timeout 600 python bench.py --streams $S --steps 3 --warmup 3 --samples 4000 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('C2 streams $S', round(d['value']))" >> gpurun_out/p10/bench.txt
done
