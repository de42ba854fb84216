# Round-1 evidence: every bench line, the ncu launch list, full ncu captures of the kernels.
# Run as one gpurun call: bash tools/evidence_r01.sh   (outputs under gpurun_out/ev/)
set -x
mkdir -p gpurun_out/ev
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/ev/smoke.log 2>&1
python bench.py > gpurun_out/ev/bench_c2.json 2> gpurun_out/ev/bench_c2.err
python bench.py --precision approx --no-e2e > gpurun_out/ev/bench_c2_approx.json 2> gpurun_out/ev/bench_c2_approx.err
python bench.py --with-conditioner --no-e2e > gpurun_out/ev/bench_c2_cond.json 2> gpurun_out/ev/bench_c2_cond.err
python bench.py --workload C3 --steps 3 --cpu-samples 8000 > gpurun_out/ev/bench_c3.json 2> gpurun_out/ev/bench_c3.err
python bench.py --workload C4 --steps 2 --cpu-samples 1600 > gpurun_out/ev/bench_c4.json 2> gpurun_out/ev/bench_c4.err
python bench.py --workload C4 --steps 2 --cpu-samples 1600 --precision tf32 --no-e2e > gpurun_out/ev/bench_c4_tf32.json 2> gpurun_out/ev/bench_c4_tf32.err
python bench.py --workload C5 --samples 8000 --steps 2 --cpu-samples 1600 --no-e2e > gpurun_out/ev/bench_c5.json 2> gpurun_out/ev/bench_c5.err
python bench.py --impl reference --steps 3 > gpurun_out/ev/bench_ref.json 2> gpurun_out/ev/bench_ref.err
python tools/bench_logits.py > gpurun_out/ev/logits.json 2>&1
python tools/sweep_layers.py > gpurun_out/ev/sweep.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ev/launches_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_cluster -c 1 -o gpurun_out/ev/cluster_c2 python tools/ncu_c2.py --n 16000 > gpurun_out/ev/ncu_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_cluster -c 1 -o gpurun_out/ev/cluster_c3 python tools/ncu_c2.py --n 2000 --layers 40 > gpurun_out/ev/ncu_c3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_batch -c 1 -o gpurun_out/ev/batch_c4 python bench.py --workload C4 --samples 200 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ev/ncu_c4.log 2>&1
ncu --set full --clock-control none -k regex:k_layer -c 1 -o gpurun_out/ev/parallel_c2 python tools/bench_logits.py > gpurun_out/ev/ncu_par.log 2>&1
ncu --set full --clock-control none -k regex:k_batch -c 1 -o gpurun_out/ev/batch_c5 python bench.py --workload C5 --samples 100 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ev/ncu_c5.log 2>&1
