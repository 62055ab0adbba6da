# texel / delta planes instead of interleaved pairs in shared memory: tests + A/B (C2, C5 16 views, C1, C3)
mkdir -p gpurun_out/pl
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pl/gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pl/gputest.log
V=paper_2107_12672_b200/_variants
for rep in 1 2 3; do
for L in product pairs; do
  if [ $L = product ]; then unset DDVR_LIB; else export DDVR_LIB=$V/libddvr_$L.so; fi
  for C in C2 C1 C3; do
    timeout 300 python bench.py --config $C --steps 20 --warmup 5 --no-extras --no-cpu-baseline > gpurun_out/pl/${C}_${L}_$rep.json 2> gpurun_out/pl/${C}_${L}_$rep.err; echo "$C $L rc=$?"
  done
  timeout 600 python bench.py --config C5 --views 16 --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/pl/C5_${L}_$rep.json 2> gpurun_out/pl/C5_${L}_$rep.err; echo "C5 $L rc=$?"
done
done
unset DDVR_LIB
python - <<'PY'
import json, glob, collections
agg = collections.defaultdict(list)
for f in sorted(glob.glob("gpurun_out/pl/*.json")):
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    k = "_".join(f.split("/")[-1].split("_")[:2])
    agg[k].append(round(d["value"] / 1e9, 2))
for k, v in sorted(agg.items()):
    print(k, v, "median", sorted(v)[len(v) // 2])
PY
