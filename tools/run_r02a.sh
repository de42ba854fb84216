# round 2, first GPU pass: tests + C2 bench + one-cluster-per-stream sweep
set -x
mkdir -p gpurun_out/r2a
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2a/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2a/pytest_gpu.log 2>&1
timeout 300 python bench.py > gpurun_out/r2a/bench_c2.json 2> gpurun_out/r2a/bench_c2.err
for S in 2 4 8 10 12 16; do
  timeout 300 python bench.py --streams $S --steps 3 --no-cpu --no-e2e > gpurun_out/r2a/bench_c2_s$S.json 2> gpurun_out/r2a/bench_c2_s$S.err
  timeout 300 python bench.py --streams $S --steps 3 --no-cpu --no-e2e --kernel tc > gpurun_out/r2a/bench_c2_tc_s$S.json 2> gpurun_out/r2a/bench_c2_tc_s$S.err
done
