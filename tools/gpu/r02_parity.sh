set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest2.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r02_gputest2.log
timeout 600 python bench.py > gpurun_out/r02_bench_c4_b.json 2> gpurun_out/r02_bench_c4_b.err; echo "bench rc=$?"
python -c "import json;d=json.loads([l for l in open('gpurun_out/r02_bench_c4_b.json') if l.startswith('{')][-1]);print('RESULT', d['value']/1e9, d['ms_per_step'], d['e2e']['value']/1e9, d['tape_free']['value']/1e9, d['sparse_state']['value']/1e9, d['clocks'])"
