# end-of-session record: full GPU suite, smoke, bench lines of every config (atomics roofline)
mkdir -p gpurun_out/last
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/last/gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/last/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/last/smoke.log
timeout 900 python bench.py > gpurun_out/last/bench_C4.json 2> gpurun_out/last/bench_C4.err; echo "C4 rc=$?"
for C in C1 C2 C3 C5; do timeout 1200 python bench.py --config $C > gpurun_out/last/bench_$C.json 2> gpurun_out/last/bench_$C.err; echo "$C rc=$?"; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/last/bench_ref.json 2> gpurun_out/last/bench_ref.err; echo "ref rc=$?"
