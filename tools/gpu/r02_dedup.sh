set -x
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_step_config.py -x -q > gpurun_out/r02_dedup_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02_dedup_tests.log
run() { timeout 300 python bench.py --no-extras --no-cpu-baseline --steps 5 --warmup 3 "$@" 2>&1 | grep '^{' | python -c "import json,sys;d=json.loads(sys.stdin.read());print('RESULT', '${DDVR_LIB##*/}', sys.argv[1:], round(d['value']/1e9,1), round(d['ms_per_step'],2), round(d['kernels']['fused_forward_adjoint']['ms'],2))" "$@"; }
run
run --split-walk
export DDVR_LIB=paper_2107_12672_b200/_variants/libddvr_nodedup.so; run; unset DDVR_LIB
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:int\)1, \(bool\)1>' -c 1 -o gpurun_out/r02_c4_dedup python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/r02_ncu_dedup.log 2>&1; echo "ncu rc=$?"
