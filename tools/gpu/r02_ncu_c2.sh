mkdir -p gpurun_out/nc2
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dvr_adjoint_kernel -c 1 -o gpurun_out/nc2/c2 python bench.py --config C2 --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/nc2/ncu.log 2>&1; echo "ncu rc=$?"
