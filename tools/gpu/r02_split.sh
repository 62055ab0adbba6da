# A/B of the split band-tape step (march + walk kernels) vs the fused kernel, + GPU tests
set -x
timeout 900 python -m pytest tests/test_gpu_step.py -x -q > gpurun_out/r02_split_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02_split_tests.log
for v in "" m4w5 m5w6; do
  if [ -n "$v" ]; then export DDVR_LIB=paper_2107_12672_b200/_variants/libddvr_$v.so; else unset DDVR_LIB; fi
  timeout 300 python bench.py --no-extras --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r02_split_$v.json 2>&1; echo "bench $v rc=$?"
  python -c "import json,sys;d=json.loads([l for l in open('gpurun_out/r02_split_$v.json') if l.startswith('{')][-1]);print('$v', d['value']/1e9, d['ms_per_step'], d['clocks'])"
done
unset DDVR_LIB
timeout 300 python bench.py --no-extras --no-cpu-baseline --fused-walk > gpurun_out/r02_split_fusedwalk.json 2>&1
python -c "import json,sys;d=json.loads([l for l in open('gpurun_out/r02_split_fusedwalk.json') if l.startswith('{')][-1]);print('fusedwalk', d['value']/1e9, d['ms_per_step'])"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:dvr_band' -c 2 -o gpurun_out/r02_c4_split python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/r02_ncu_split.log 2>&1; echo "ncu rc=$?"
