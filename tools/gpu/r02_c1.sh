set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c1_launches.csv python bench.py --config C1 --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/r02_c1_launch.log 2>&1; echo "launch rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:dvr_adjoint' -c 1 -o gpurun_out/r02_c1 python bench.py --config C1 --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/r02_ncu_c1.log 2>&1; echo "ncu rc=$?"
timeout 300 python bench.py --config C1 --graph --no-cpu-baseline > gpurun_out/r02_bench_C1_graph.json 2>&1; echo "graph rc=$?"
