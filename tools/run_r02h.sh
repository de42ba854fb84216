set -x
mkdir -p gpurun_out/r2h
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2h/build.log 2>&1
timeout 2400 bash tools/diag_c2.sh "base DVW_CHAIN0=0 DVW_DEADFLAG=0 DVW_SKIPSTAGE=0 DVW_CHAIN0=0,DVW_DEADFLAG=0,DVW_SKIPSTAGE=0 DVW_CHAIN0=0,DVW_DEADFLAG=0,DVW_SKIPSTAGE=0,DVW_EXP=0 base" gpurun_out/r2h > gpurun_out/r2h/diag.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "watchdog" > gpurun_out/r2h/pytest_wd.log 2>&1
