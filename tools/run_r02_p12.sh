mkdir -p gpurun_out/p12
for LP in 3 4; do
  DVW_CLUSTER_LP=$LP timeout 600 python bench.py --streams 56 --steps 3 --warmup 3 --samples 4000 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('C2 x56 LP $LP', round(d['value']), d['config']['grid'])" >> gpurun_out/p12/bench.txt
done
for W in 4 6; do
  DVW_CLUSTER_W=$W timeout 600 python bench.py --streams $((7*W)) --steps 3 --warmup 3 --samples 4000 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('C2 x$((7*W)) W $W', round(d['value']), d['config']['grid'])" >> gpurun_out/p12/bench.txt
done
cat gpurun_out/p12/bench.txt
