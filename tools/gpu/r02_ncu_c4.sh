# ncu --set full of the fused C4 kernel (ROLE 1, band tape) at bench.py's fixed dense state
set -x
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:int\)1, \(bool\)1>' -c 1 -o gpurun_out/r02_c4_dense \
  python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/r02_ncu_c4.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/r02_ncu_c4.log
