# round 2 GPU pass g: chain CTA 0 with the per-code layer-0 table (chain0_*): parity + timing
set -x
mkdir -p gpurun_out/r2g
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2g/smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "cluster or free_running or c2_full or appc or approx or quantized or determinism or causality or zero_weights or edge or session or auto" > gpurun_out/r2g/pytest_cl.log 2>&1
timeout 300 python tools/sweep_layers.py --layers 1,2,3,4,8,20,40 --n 8000 > gpurun_out/r2g/sweep.txt 2>&1
timeout 300 python bench.py --no-cpu > gpurun_out/r2g/bench_c2.json 2> gpurun_out/r2g/bench_c2.err
timeout 300 python tools/trace_c2.py > gpurun_out/r2g/trace_c2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "tc or batched or shard or sampler or watchdog" > gpurun_out/r2g/pytest_tc.log 2>&1
timeout 600 python bench.py --workload C4 --no-cpu > gpurun_out/r2g/bench_c4.json 2> gpurun_out/r2g/bench_c4.err
timeout 600 python bench.py --workload C5 --samples 8000 --no-cpu --steps 3 > gpurun_out/r2g/bench_c5.json 2> gpurun_out/r2g/bench_c5.err
for t in synccheck racecheck; do
  timeout 400 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_tiny.py --kernel cluster > gpurun_out/r2g/san_cluster_$t.log 2>&1; echo "exit $?" >> gpurun_out/r2g/san_cluster_$t.log
done
