# round 2 final evidence: full GPU tests, bench lines (C2 default, C3, C4, C5 per-rank), launch list, sanitizers
set -x
mkdir -p gpurun_out/r2q
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2q/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2q/pytest_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/r2q/bench_c2.json 2> gpurun_out/r2q/bench_c2.err
timeout 900 python bench.py --workload C3 --no-cpu > gpurun_out/r2q/bench_c3.json 2> gpurun_out/r2q/bench_c3.err
timeout 900 python bench.py --workload C4 --no-cpu > gpurun_out/r2q/bench_c4.json 2> gpurun_out/r2q/bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2q/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/r2q/bench_under_ncu.log 2>&1
for k in cluster stream tc parallel conditioner; do
  for t in memcheck racecheck synccheck; do
    timeout 400 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_tiny.py --kernel $k > gpurun_out/r2q/san_${k}_${t}.log 2>&1
    echo "exit $?" >> gpurun_out/r2q/san_${k}_${t}.log
  done
done
