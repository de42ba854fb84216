set -x
mkdir -p gpurun_out/r2p
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2p/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "balanced" > gpurun_out/r2p/pytest_bal.log 2>&1
LAYERS=20 timeout 1500 bash tools/diag_c2.sh "base DVW_EXP=10 base DVW_EXP=10" gpurun_out/r2p > gpurun_out/r2p/diag.log 2>&1
