set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest5.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_gputest5.log
grep -B 20 "Error" gpurun_out/r02_gputest5.log | head -40
cat > /tmp/detbench.py <<'PY'
import sys, json, torch, numpy as np
sys.path.insert(0, '.')
import bench
PY
run() { timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 3 --warmup 3 "$@" 2>&1 | grep '^{' | python -c "import json,sys;d=json.loads(sys.stdin.read());print('RESULT', sys.argv[1:], round(d['value']/1e9,2), round(d['ms_per_step'],3))" "$@"; }
run --config C4
