set -x
mkdir -p gpurun_out/r2k
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2k/build.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_cluster -c 1 -o gpurun_out/r2k/cluster_c2 python tools/ncu_c2.py --n 3000 > gpurun_out/r2k/ncu_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2k/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/r2k/bench_under_ncu.log 2>&1
ncu -i gpurun_out/r2k/cluster_c2.ncu-rep --page source --csv > gpurun_out/r2k/cluster_source.csv 2>/dev/null
ncu -i gpurun_out/r2k/cluster_c2.ncu-rep --page raw --csv > gpurun_out/r2k/cluster_raw.csv 2>/dev/null
ncu -i gpurun_out/r2k/cluster_c2.ncu-rep --page details --csv > gpurun_out/r2k/cluster_details.csv 2>/dev/null
