run() { timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 5 --warmup 3 "$@" 2>&1 | grep '^{' | python -c "import json,sys;d=json.loads(sys.stdin.read());print('RESULT', sys.argv[1:], round(d['value']/1e9,2), round(d['ms_per_step'],3), d['kernels'])" "$@"; }
run --config C3; run --config C3 --fused; run --config C3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_properties.py tests/test_gpu_smoke.py -x -q > gpurun_out/r02_c3_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02_c3_tests.log
