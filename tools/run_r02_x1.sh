# AUTO crossover: multi-stream cluster kernel vs batched TC kernel at C2 and C5 shapes
mkdir -p gpurun_out/x1
for S in 128 256 448 896; do for K in cluster tc; do
  timeout 600 python bench.py --streams $S --steps 3 --warmup 3 --samples 1000 --no-cpu --no-e2e --kernel $K 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('C2 streams $S $K', round(d['value']), d['config']['grid'], d['config']['launches_per_step'])" >> gpurun_out/x1/x.txt
done; done
for G in 4 3 2; do for K in cluster tc; do
  timeout 900 python bench.py --workload C5 --samples 1000 --as-shard-of $G --steps 3 --warmup 3 --no-cpu --no-e2e --kernel $K 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('C5 shard-of $G $K', d['config']['streams_per_gpu'], round(d['value']), d['config']['grid'], d['config']['launches_per_step'])" >> gpurun_out/x1/x.txt
done; done
cat gpurun_out/x1/x.txt
