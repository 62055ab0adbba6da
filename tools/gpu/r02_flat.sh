mkdir -p gpurun_out/fl
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fl/gputest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fl/gputest.log
for rep in 1 2 3; do timeout 300 python bench.py --config C1 --steps 20 --warmup 5 --no-extras --no-cpu-baseline > gpurun_out/fl/C1_$rep.json 2>/dev/null; echo "C1 rc=$?"; done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/fl/*.json")):
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    print(f.split("/")[-1], round(d["value"] / 1e9, 3), round(d["ms_per_step"], 4), d.get("gpu_launches"))
PY
