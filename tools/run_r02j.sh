set -x
mkdir -p gpurun_out/r2j
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2j/smoke.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "watchdog" > gpurun_out/r2j/pytest_wd.log 2>&1
timeout 300 python tools/sweep_layers.py --layers 1,20,40 --n 8000 > gpurun_out/r2j/sweep.txt 2>&1
timeout 600 python bench.py > gpurun_out/r2j/bench_c2.json 2> gpurun_out/r2j/bench_c2.err
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2j/pytest_all.log 2>&1
timeout 600 python bench.py --workload C3 --no-cpu > gpurun_out/r2j/bench_c3.json 2> gpurun_out/r2j/bench_c3.err
