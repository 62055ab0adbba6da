run() { timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 3 --warmup 3 "$@" 2>&1 | grep '^{' | python -c "import json,sys;d=json.loads(sys.stdin.read());print('RESULT', '${DDVR_LIB##*/}', sys.argv[1:], round(d['value']/1e9,2), round(d['ms_per_step'],3))" "$@"; }
run --config C5 --views 16; run --config C2
export DDVR_LIB=paper_2107_12672_b200/_variants/libddvr_nolds.so; run --config C5 --views 16; run --config C2
