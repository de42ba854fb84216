# Round-2 final evidence: bench lines of every workload, the ncu launch list of the headline, full ncu
# captures of the multi-stream cluster kernel.  One gpurun call: bash tools/evidence_r02.sh (gpurun_out/ev2/)
set -x
mkdir -p gpurun_out/ev2
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/ev2/smoke.log 2>&1
python bench.py > gpurun_out/ev2/bench_c2.json 2> gpurun_out/ev2/bench_c2.err
python bench.py --workload C1 --steps 5 > gpurun_out/ev2/bench_c1.json 2> gpurun_out/ev2/bench_c1.err
python bench.py --workload C3 --steps 3 --cpu-samples 8000 > gpurun_out/ev2/bench_c3.json 2> gpurun_out/ev2/bench_c3.err
python bench.py --streams 56 --steps 3 --no-cpu > gpurun_out/ev2/bench_c2_s56.json 2> gpurun_out/ev2/bench_c2_s56.err
python bench.py --workload C4 --steps 2 --cpu-samples 1600 > gpurun_out/ev2/bench_c4.json 2> gpurun_out/ev2/bench_c4.err
python bench.py --workload C5 --as-shard-of 8 --steps 3 --cpu-samples 1600 --no-e2e > gpurun_out/ev2/bench_c5_g8_full.json 2> gpurun_out/ev2/bench_c5_g8_full.err
python bench.py --workload C5 --samples 8000 --steps 3 --no-cpu --no-e2e > gpurun_out/ev2/bench_c5_g1_8k.json 2> gpurun_out/ev2/bench_c5_g1_8k.err
python bench.py --impl reference --steps 3 > gpurun_out/ev2/bench_ref.json 2> gpurun_out/ev2/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev2/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ev2/launches_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_cluster -c 1 -o gpurun_out/ev2/cluster_c2_s56 python bench.py --streams 56 --samples 500 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ev2/ncu_c2_s56.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_cluster -c 1 -o gpurun_out/ev2/cluster_c5_s256 python bench.py --workload C5 --as-shard-of 8 --samples 200 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ev2/ncu_c5_s256.log 2>&1
