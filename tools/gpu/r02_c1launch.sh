# C1 launch list (graph replay) + C2/C3 for where small-config time goes
mkdir -p gpurun_out/c1l
timeout 300 python bench.py --config C1 --no-extras --no-cpu-baseline > gpurun_out/c1l/C1.json 2> gpurun_out/c1l/C1.err; echo "C1 rc=$?"
timeout 300 python bench.py --config C1 --graph off --no-extras --no-cpu-baseline > gpurun_out/c1l/C1_nograph.json 2>&1; echo "C1 nograph rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c1l/launches_C1.csv python bench.py --config C1 --steps 2 --warmup 3 --graph off --no-extras --no-cpu-baseline > gpurun_out/c1l/ncu.log 2>&1; echo "ncu rc=$?"
