set -x
mkdir -p gpurun_out/ev
python bench.py > gpurun_out/ev/bench_c2.json 2> gpurun_out/ev/bench_c2.err
python bench.py --workload C3 --steps 3 --cpu-samples 8000 > gpurun_out/ev/bench_c3.json 2> gpurun_out/ev/bench_c3.err
python bench.py --workload C4 --steps 2 --cpu-samples 1600 > gpurun_out/ev/bench_c4.json 2> gpurun_out/ev/bench_c4.err
python bench.py --workload C5 --samples 8000 --steps 2 --cpu-samples 1600 --no-e2e > gpurun_out/ev/bench_c5.json 2> gpurun_out/ev/bench_c5.err
python bench.py --impl reference --steps 3 > gpurun_out/ev/bench_ref.json 2> gpurun_out/ev/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ev/launches_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_cluster -c 1 -o gpurun_out/ev/cluster_c2 python tools/ncu_c2.py --n 3000 > gpurun_out/ev/ncu_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_cluster -c 1 -o gpurun_out/ev/cluster_c3 python tools/ncu_c2.py --n 2000 --layers 40 > gpurun_out/ev/ncu_c3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_batch -c 1 -o gpurun_out/ev/batch_c4 python bench.py --workload C4 --samples 200 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ev/ncu_c4.log 2>&1
