# round 2, second GPU pass: full GPU tests, floor probe, trace, bench, ncu C2, sanitizers
set -x
mkdir -p gpurun_out/r2b
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2b/pytest_gpu.log 2>&1
python -c "from paper_1702_07825_b200._lib import measure_floor; import json; [print(json.dumps(measure_floor(0))) for _ in range(3)]" > gpurun_out/r2b/floor.log 2>&1
timeout 300 python tools/trace_c2.py > gpurun_out/r2b/trace_c2.log 2>&1
timeout 300 python bench.py > gpurun_out/r2b/bench_c2.json 2> gpurun_out/r2b/bench_c2.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_cluster -c 1 -o gpurun_out/r2b/cluster_c2 python tools/ncu_c2.py --n 16000 > gpurun_out/r2b/ncu_c2.log 2>&1
for k in cluster stream tc parallel conditioner; do
  for t in memcheck racecheck synccheck; do
    timeout 600 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_tiny.py --kernel $k > gpurun_out/r2b/san_${k}_${t}.log 2>&1
    echo "exit $?" >> gpurun_out/r2b/san_${k}_${t}.log
  done
done
