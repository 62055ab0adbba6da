mkdir -p gpurun_out/e4
V=paper_2107_12672_b200/_variants
for rep in 1 2; do
for L in product eu4; do
  if [ $L = product ]; then unset DDVR_LIB; else export DDVR_LIB=$V/libddvr_$L.so; fi
  timeout 600 python bench.py --config C5 --views 16 --no-extras --no-cpu-baseline > gpurun_out/e4/C5_${L}_$rep.json 2>/dev/null; echo "C5 $L rc=$?"
  timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-extras --no-cpu-baseline > gpurun_out/e4/C2_${L}_$rep.json 2>/dev/null; echo "C2 $L rc=$?"
done
done
unset DDVR_LIB
python - <<'PY'
import json, glob, collections
agg = collections.defaultdict(list)
for f in sorted(glob.glob("gpurun_out/e4/*.json")):
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    k = "_".join(f.split("/")[-1].split("_")[:2])
    agg[k].append(round(d["value"] / 1e9, 2))
for k, v in sorted(agg.items()):
    print(k, v)
PY
