mkdir -p gpurun_out/nc1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:fold_cells|prior_volume|pack_cells|tf_slots|adam_kernel|finite_check" -c 8 -o gpurun_out/nc1/c1small python bench.py --config C1 --steps 1 --warmup 3 --graph off --no-extras --no-cpu-baseline > gpurun_out/nc1/ncu.log 2>&1; echo "ncu rc=$?"
