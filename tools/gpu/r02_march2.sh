set -x
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_step_config.py tests/test_gpu_checked.py -x -q > gpurun_out/r02_m2_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02_m2_tests.log
run() { timeout 300 python bench.py --no-extras --no-cpu-baseline --steps 5 --warmup 3 "$@" 2>&1 | grep '^{' | python -c "import json,sys;d=json.loads(sys.stdin.read());print('RESULT', sys.argv[1:], round(d['value']/1e9,1), round(d['ms_per_step'],2), round(d['kernels']['fused_forward_adjoint']['ms'],2))" "$@"; }
run
run
run --split-walk
