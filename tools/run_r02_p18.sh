mkdir -p gpurun_out/p18
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for SP in 0 1 0 1; do
 DVW_SKIP_SPREAD=$SP timeout 600 python tools/sweep_layers.py --layers 20 --n 8000 2>&1 | tail -1 | sed "s/^/spread $SP batch-1 /" >> gpurun_out/p18/bench.txt
 DVW_SKIP_SPREAD=$SP timeout 600 python bench.py --streams 56 --steps 3 --warmup 3 --samples 4000 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('spread $SP C2 x56', round(d['value']), d['config']['cluster_ctas'])" >> gpurun_out/p18/bench.txt
done
DVW_SKIP_SPREAD=1 timeout 600 python tools/pipe_check.py > gpurun_out/p18/pipe_check.log 2>&1
DVW_SKIP_SPREAD=1 timeout 900 python -m pytest tests -m gpu -x -q -k "cluster" > gpurun_out/p18/tests_cluster.txt 2>&1
