set -x
mkdir -p gpurun_out/p5
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p5/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "multi_stream" > gpurun_out/p5/tests_ms.txt 2>&1
timeout 600 python tools/pipe_check.py > gpurun_out/p5/pipe_check.log 2>&1
for XS in "3 4" "3 2"; do set -- $XS
  DVW_XPB=$1 DVW_XSB=$2 timeout 600 python bench.py --streams 56 --steps 3 --samples 2000 --no-cpu --no-e2e --kernel cluster 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('xpb $1 xsb $2 C2x56', round(d['value']))" >> gpurun_out/p5/bench.txt
  DVW_XPB=$1 DVW_XSB=$2 timeout 600 python bench.py --workload C5 --samples 1000 --as-shard-of 8 --steps 3 --no-cpu --no-e2e --kernel cluster 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('xpb $1 xsb $2 C5x256', round(d['value']))" >> gpurun_out/p5/bench.txt
done
timeout 900 python bench.py --workload C5 --samples 1000 --steps 3 --no-cpu --no-e2e --kernel cluster 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('C5x2048 cluster', round(d['value']), d['config']['grid'])" >> gpurun_out/p5/bench.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p5/gpu_tests.txt 2>&1
