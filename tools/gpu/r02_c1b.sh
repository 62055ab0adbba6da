set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest3.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_gputest3.log
timeout 300 python bench.py --config C1 > gpurun_out/r02_bench_C1b.json 2>&1; echo "c1 rc=$?"
grep '^{' gpurun_out/r02_bench_C1b.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print('RESULT C1', d['value']/1e9, d['ms_per_step'], d['e2e']['value']/1e9, d['gpu_launches'], d['config']['step'], d['clocks'])"
timeout 300 python bench.py --config C2 --no-cpu-baseline > gpurun_out/r02_bench_C2b.json 2>&1; echo "c2 rc=$?"
grep '^{' gpurun_out/r02_bench_C2b.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print('RESULT C2', d['value']/1e9, d['ms_per_step'], d['e2e']['value']/1e9)"
