timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_step.py -x -q 2>&1 | tail -2
run() { timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 3 --warmup 3 "$@" 2>&1 | grep '^{' | python -c "import json,sys;d=json.loads(sys.stdin.read());print('RESULT', sys.argv[1:], round(d['value']/1e9,2), round(d['ms_per_step'],3))" "$@"; }
run --config C5 --views 16; run --config C4; run --config C4 --deterministic; run --config C5 --views 16 --deterministic
