# round 2 GPU pass f: batched lo-on-chip (tests + C4/C5 bench), watchdog under memcheck, sanitizers
set -x
mkdir -p gpurun_out/r2f
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2f/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "tc or batched or session or shard or sampler or quantized or auto" > gpurun_out/r2f/pytest_tc.log 2>&1
timeout 600 python bench.py --workload C4 --no-cpu > gpurun_out/r2f/bench_c4.json 2> gpurun_out/r2f/bench_c4.err
timeout 600 python bench.py --workload C5 --samples 8000 --no-cpu --steps 3 > gpurun_out/r2f/bench_c5.json 2> gpurun_out/r2f/bench_c5.err
timeout 300 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k watchdog > gpurun_out/r2f/san_watchdog.log 2>&1
for k in cluster stream tc parallel conditioner; do
  for t in memcheck synccheck racecheck; do
    timeout 400 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_tiny.py --kernel $k > gpurun_out/r2f/san_${k}_${t}.log 2>&1
    echo "exit $?" >> gpurun_out/r2f/san_${k}_${t}.log
  done
done
