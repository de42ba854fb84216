mkdir -p gpurun_out/p15
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/p15/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p15/gpu_tests.txt 2>&1
timeout 600 python tools/pipe_check.py > gpurun_out/p15/pipe_check.log 2>&1
for a in "56 400" "14 400" "56 2000" "28 400" "9 300"; do timeout 120 python tools/ptcheck_tmp.py $a >> gpurun_out/p15/ptcheck.txt 2>&1; done
timeout 600 python bench.py --streams 56 --steps 3 --warmup 3 --samples 4000 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('C2 streams 56', round(d['value']))" >> gpurun_out/p15/bench.txt
(cd ab/1 && python tools/ptrace_pipe.py > /root/repo/gpurun_out/p15/pt.txt 2>&1; PT_STREAMS=28 python tools/ptrace_pipe.py >> /root/repo/gpurun_out/p15/pt.txt 2>&1; PT_CFG=C3 python tools/ptrace_pipe.py >> /root/repo/gpurun_out/p15/pt.txt 2>&1)
