# view groups as the default (4): tests + A/B against DDVR_VGROUP=1 on C4, C4 tape-free, C5, C2, C3
mkdir -p gpurun_out/vg2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/vg2/gputest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/vg2/gputest.log
for rep in 1 2; do
for G in 4 1; do
  DDVR_VGROUP=$G timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/vg2/C4_g${G}_$rep.json 2>/dev/null; echo "C4 $G rc=$?"
  DDVR_VGROUP=$G timeout 600 python bench.py --no-band-tape --no-extras --no-cpu-baseline > gpurun_out/vg2/C4nt_g${G}_$rep.json 2>/dev/null; echo "C4nt $G rc=$?"
  DDVR_VGROUP=$G timeout 600 python bench.py --config C5 --views 16 --no-extras --no-cpu-baseline > gpurun_out/vg2/C5_g${G}_$rep.json 2>/dev/null; echo "C5 $G rc=$?"
  DDVR_VGROUP=$G timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-extras --no-cpu-baseline > gpurun_out/vg2/C2_g${G}_$rep.json 2>/dev/null; echo "C2 $G rc=$?"
done
done
python - <<'PY'
import json, glob, collections
agg = collections.defaultdict(list)
for f in sorted(glob.glob("gpurun_out/vg2/*.json")):
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    k = "_".join(f.split("/")[-1].split("_")[:2])
    agg[k].append(round(d["value"] / 1e9, 2))
for k, v in sorted(agg.items()):
    print(k, v)
PY
