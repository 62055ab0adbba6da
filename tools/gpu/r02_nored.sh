set -x
run() { timeout 300 python bench.py --no-extras --no-cpu-baseline --steps 5 --warmup 3 "$@" 2>&1 | grep '^{' | python -c "import json,sys;d=json.loads(sys.stdin.read());print('RESULT', sys.argv[1:], round(d['value']/1e9,1), round(d['ms_per_step'],2), d['kernels'])" "$@"; }
run
run --fused-walk
export DDVR_LIB=paper_2107_12672_b200/_variants/libddvr_nored.so
run
run --fused-walk
