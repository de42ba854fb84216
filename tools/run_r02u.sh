set -x
mkdir -p gpurun_out/r2u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2u/build.log 2>&1
timeout 600 python tools/pipe_check.py > gpurun_out/r2u/pipe_check.log 2>&1
