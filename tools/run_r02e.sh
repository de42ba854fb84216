# round 2 GPU pass e: cluster-kernel experiments (DVW_EXP) and the watchdog test
set -x
mkdir -p gpurun_out/r2e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2e/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "watchdog" > gpurun_out/r2e/pytest_sel.log 2>&1
timeout 1500 bash tools/diag_c2.sh "0 e1 e2 e4 e3 e7 0" gpurun_out/r2e > gpurun_out/r2e/diag.log 2>&1
