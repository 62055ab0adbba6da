mkdir -p gpurun_out/c3f
for rep in 1 2 3; do
for M in default fused; do
  X=""; [ $M = fused ] && X="--fused"
  timeout 300 python bench.py --config C3 --steps 20 --warmup 5 $X --no-extras --no-cpu-baseline > gpurun_out/c3f/C3_${M}_$rep.json 2>/dev/null; echo "C3 $M rc=$?"
done
done
python - <<'PY'
import json, glob, collections
agg = collections.defaultdict(list)
for f in sorted(glob.glob("gpurun_out/c3f/*.json")):
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    k = "_".join(f.split("/")[-1].split("_")[:2])
    agg[k].append(round(d["value"] / 1e9, 2))
for k, v in sorted(agg.items()):
    print(k, v)
PY
