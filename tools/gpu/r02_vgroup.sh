# view groups (CTAs cycle over similar views per tile) for L2 sharing of the ray tubes: C4
mkdir -p gpurun_out/vg
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/vg/gputest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/vg/gputest.log
for rep in 1 2; do
  timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/vg/C4_base_$rep.json 2>/dev/null; echo "base rc=$?"
  timeout 600 python bench.py --sort-views --no-extras --no-cpu-baseline > gpurun_out/vg/C4_sorted_$rep.json 2>/dev/null; echo "sorted rc=$?"
  for G in 2 4 8; do
    DDVR_VGROUP=$G timeout 600 python bench.py --sort-views --no-extras --no-cpu-baseline > gpurun_out/vg/C4_vg${G}_$rep.json 2>/dev/null; echo "vg$G rc=$?"
  done
  DDVR_VGROUP=4 timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/vg/C4_vg4unsorted_$rep.json 2>/dev/null; echo "vg4u rc=$?"
done
python - <<'PY'
import json, glob, collections
agg = collections.defaultdict(list)
for f in sorted(glob.glob("gpurun_out/vg/*.json")):
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    k = "_".join(f.split("/")[-1].split("_")[:2])
    agg[k].append((round(d["value"] / 1e9, 2), round(d["roofline"]["launch_ms"], 2)))
for k, v in sorted(agg.items()):
    print(k, v)
PY
