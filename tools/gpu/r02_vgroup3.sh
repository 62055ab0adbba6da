mkdir -p gpurun_out/vg4
for rep in 1 2; do
for G in 4 16 64; do
  DDVR_VGROUP=$G timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/vg4/C4_g${G}_$rep.json 2>/dev/null; echo "C4 $G rc=$?"
done
for G in 4 16; do
  DDVR_VGROUP=$G timeout 600 python bench.py --config C5 --views 16 --no-extras --no-cpu-baseline > gpurun_out/vg4/C5_g${G}_$rep.json 2>/dev/null; echo "C5 $G rc=$?"
done
done
python - <<'PY'
import json, glob, collections
agg = collections.defaultdict(list)
for f in sorted(glob.glob("gpurun_out/vg4/*.json")):
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    k = "_".join(f.split("/")[-1].split("_")[:2])
    agg[k].append(round(d["value"] / 1e9, 2))
for k, v in sorted(agg.items()):
    print(k, v)
PY
