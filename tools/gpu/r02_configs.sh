# bench lines of every config at the fixed state + ncu of each config's dominant kernel
set -x
for C in C1 C2 C3 C5; do
  timeout 900 python bench.py --config $C > gpurun_out/r02_bench_$C.json 2> gpurun_out/r02_bench_$C.err; echo "bench $C rc=$?"
  python -c "import json;d=json.loads([l for l in open('gpurun_out/r02_bench_$C.json') if l.startswith('{')][-1]);print('RESULT $C', d['value']/1e9, d['ms_per_step'], (d.get('e2e') or {}).get('value',0)/1e9, d['kernels'], d['clocks'])"
done
K='--kernel-name-base demangled'
timeout 900 ncu --set full --clock-control none --import-source on $K -k 'regex:dvr_adjoint_kernel' -c 2 -o gpurun_out/r02_c5_v16 python bench.py --config C5 --views 16 --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/r02_ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on $K -k 'regex:dvr_adjoint_kernel' -c 2 -o gpurun_out/r02_c2 python bench.py --config C2 --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/r02_ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on $K -k 'regex:dvr_adjoint_kernel|dvr_forward_kernel' -c 4 -o gpurun_out/r02_c3 python bench.py --config C3 --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/r02_ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
