set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02_gputest.log
timeout 600 python bench.py > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r02_bench_c4.json; tail -5 gpurun_out/r02_bench_c4.err
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:dvr_adjoint_kernel<8, 1, 1, 1>" -c 1 -o gpurun_out/r02_c4_dense python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/r02_ncu_c4.log 2>&1; echo "ncu rc=$?"
tail -5 gpurun_out/r02_ncu_c4.log
