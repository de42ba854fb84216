# round 2 GPU pass c: build, smoke, full gpu tests, C2 bench, floor probe, small-batch sweep
set -x
mkdir -p gpurun_out/r2c
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2c/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2c/pytest_gpu.log 2>&1
timeout 300 python bench.py > gpurun_out/r2c/bench_c2.json 2> gpurun_out/r2c/bench_c2.err
timeout 120 python -c "from paper_1702_07825_b200._lib import measure_floor; import json; [print(json.dumps(measure_floor(0))) for _ in range(3)]" > gpurun_out/r2c/floor.log 2>&1
for S in 2 4 8 16; do
  timeout 300 python bench.py --streams $S --steps 3 --no-cpu --no-e2e > gpurun_out/r2c/bench_c2_s$S.json 2> gpurun_out/r2c/bench_c2_s$S.err
  timeout 300 python bench.py --streams $S --steps 3 --no-cpu --no-e2e --kernel tc > gpurun_out/r2c/bench_c2_tc_s$S.json 2> gpurun_out/r2c/bench_c2_tc_s$S.err
done
timeout 600 python bench.py --workload C4 --no-cpu > gpurun_out/r2c/bench_c4.json 2> gpurun_out/r2c/bench_c4.err
