set -x
mkdir -p gpurun_out/r2i
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2i/build.log 2>&1
timeout 300 python tools/sweep_layers.py --layers 20,40 --n 8000 > gpurun_out/r2i/sweep_base.txt 2>&1
DVW_PAD_CLUSTERS=10 timeout 300 python tools/sweep_layers.py --layers 20,40 --n 8000 > gpurun_out/r2i/sweep_pad10.txt 2>&1
timeout 2400 bash tools/diag_c2.sh "DVW_CHAIN0=0 DVW_BAR_ALIGNED=0 DVW_CHAIN0=0,DVW_BAR_ALIGNED=0 DVW_DEADFLAG=0 DVW_EXP=0" gpurun_out/r2i > gpurun_out/r2i/diag.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "watchdog or cluster or c2_full or session" > gpurun_out/r2i/pytest.log 2>&1
