# round-2 measurements of record: bench lines of every config, fixed-state reproducibility,
# the C4 launch list; ncu --set full of each config's dominant kernel at the timed state
# (reports stay in /tmp on the box; their raw pages come back as CSV)
set -x
mkdir -p gpurun_out/final /tmp/ncu
if [ "$1" = bench ]; then
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/final/bench_C4.json 2> gpurun_out/final/bench_C4.err; echo "c4 rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/final/bench_C4_s20.json 2>&1; echo "c4s20 rc=$?"
for C in C1 C2 C3 C5; do timeout 1200 python bench.py --config $C > gpurun_out/final/bench_$C.json 2> gpurun_out/final/bench_$C.err; echo "$C rc=$?"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_C4.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > /dev/null 2>&1; echo "launch rc=$?"
fi
if [ "$1" = ncu ]; then
K='--set full --clock-control none --import-source on --kernel-name-base demangled'
cap() {  # name, kernel regex, count, bench args...
  n=$1; k=$2; c=$3; shift 3
  timeout 900 ncu $K -k "regex:$k" -c $c -o /tmp/ncu/$n python bench.py "$@" --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/final/ncu_$n.log 2>&1; echo "ncu $n rc=$?"
  ncu -i /tmp/ncu/$n.ncu-rep --page raw --csv > gpurun_out/final/ncu_${n}_raw.csv 2>/dev/null
}
cap C4 'int\)1, \(bool\)1, \(bool\)0, \(int\)1>' 1
cap C5 'dvr_adjoint_kernel' 1 --config C5 --views 16
cap C2 'dvr_adjoint_kernel' 1 --config C2
cap C3 'dvr_adjoint_kernel' 1 --config C3
cap C1 'dvr_adjoint_kernel' 1 --config C1 --graph off
ls -la gpurun_out/final
fi
