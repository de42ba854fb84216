# round 2 GPU pass d: fixed tests (watchdog, TC session), cluster-kernel diagnostics, trace
set -x
mkdir -p gpurun_out/r2d
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2d/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "watchdog or tc_streaming_session" > gpurun_out/r2d/pytest_sel.log 2>&1
timeout 300 python tools/trace_c2.py > gpurun_out/r2d/trace_c2.log 2>&1
timeout 1500 bash tools/diag_c2.sh "0 1 2 4 8 16 6 7 15" gpurun_out/r2d > gpurun_out/r2d/diag.log 2>&1
