set -x
timeout 900 python -m pytest tests/test_gpu_step_config.py tests/test_gpu_parity.py tests/test_api.py -x -q -m gpu > gpurun_out/r02_hold_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02_hold_tests.log
run() { timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 3 --warmup 2 "$@" 2>&1 | grep '^{' | python -c "import json,sys;d=json.loads(sys.stdin.read());print('RESULT', '${DDVR_LIB##*/}', sys.argv[1:], round(d['value']/1e9,2), round(d['ms_per_step'],3))" "$@"; }
for v in "" nohold; do
  if [ -n "$v" ]; then export DDVR_LIB=paper_2107_12672_b200/_variants/libddvr_$v.so; fi
  run --config C5 --views 16; run --config C2; run --config C1; run --config C3
done
