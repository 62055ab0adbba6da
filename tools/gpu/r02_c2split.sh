mkdir -p gpurun_out/c2s
for rep in 1 2 3; do
for K in auto 2 4; do
  timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --ray-split $K --no-extras --no-cpu-baseline > gpurun_out/c2s/C2_${K}_$rep.json 2>/dev/null; echo "C2 $K rc=$?"
done
done
python - <<'PY'
import json, glob, collections
agg = collections.defaultdict(list)
for f in sorted(glob.glob("gpurun_out/c2s/*.json")):
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    k = "_".join(f.split("/")[-1].split("_")[:2])
    agg[k].append(round(d["value"] / 1e9, 2))
for k, v in sorted(agg.items()):
    print(k, v)
PY
