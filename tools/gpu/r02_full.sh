set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_gputest4.log
timeout 600 python bench.py > gpurun_out/r02_bench_c4_c.json 2> gpurun_out/r02_bench_c4_c.err; echo "bench rc=$?"
grep '^{' gpurun_out/r02_bench_c4_c.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print('RESULT C4', d['value']/1e9, d['ms_per_step'], d['e2e']['value']/1e9, d['tape_free']['value']/1e9, d['sparse_state']['value']/1e9, d['roofline']['frac'], d['clocks'])"
timeout 600 python bench.py --config C3 --no-cpu-baseline > gpurun_out/r02_bench_C3b.json 2>&1; echo "c3 rc=$?"
grep '^{' gpurun_out/r02_bench_C3b.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print('RESULT C3', d['value']/1e9, d['ms_per_step'], d['e2e']['value']/1e9)"
