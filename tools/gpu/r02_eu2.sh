mkdir -p gpurun_out/eu
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/eu/gputest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/eu/gputest.log
for C in C3 C1 C2; do timeout 300 python bench.py --config $C --steps 20 --warmup 5 --no-extras --no-cpu-baseline > gpurun_out/eu/$C.json 2>/dev/null; echo "$C rc=$?"; done
timeout 600 python bench.py --config C5 --views 16 --no-extras --no-cpu-baseline > gpurun_out/eu/C5.json 2>/dev/null; echo "C5 rc=$?"
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/eu/*.json")):
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    print(f.split("/")[-1], round(d["value"] / 1e9, 2))
PY
