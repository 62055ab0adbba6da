# C1 launch list with the ray split, warm caches (--cache-control none)
mkdir -p gpurun_out/c1l2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/c1l2/launches_C1.csv python bench.py --config C1 --steps 2 --warmup 3 --graph off --no-extras --no-cpu-baseline > gpurun_out/c1l2/ncu.log 2>&1; echo "ncu rc=$?"
