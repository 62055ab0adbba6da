mkdir -p gpurun_out/fo2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fo2/gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/fo2/gputest.log
V=paper_2107_12672_b200/_variants
for rep in 1 2 3; do
for L in product head; do
  if [ $L = product ]; then unset DDVR_LIB; else export DDVR_LIB=$V/libddvr_$L.so; fi
  timeout 300 python bench.py --config C1 --steps 20 --warmup 5 --no-extras --no-cpu-baseline > gpurun_out/fo2/C1_${L}_$rep.json 2> gpurun_out/fo2/C1_${L}_$rep.err; echo "C1 $L rc=$?"
done
done
unset DDVR_LIB
timeout 300 python bench.py --config C4 --no-extras --no-cpu-baseline > gpurun_out/fo2/C4.json 2> gpurun_out/fo2/C4.err; echo "C4 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/fo2/launches_C1.csv python bench.py --config C1 --steps 2 --warmup 3 --graph off --no-extras --no-cpu-baseline > gpurun_out/fo2/ncu.log 2>&1; echo "ncu rc=$?"
python - <<'PY'
import json, glob, collections
agg = collections.defaultdict(list)
for f in sorted(glob.glob("gpurun_out/fo2/*.json")):
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    k = "_".join(f.split("/")[-1].split("_")[:2])
    agg[k].append(round(d["value"] / 1e9, 2))
for k, v in sorted(agg.items()):
    print(k, v, "median", sorted(v)[len(v) // 2])
PY
