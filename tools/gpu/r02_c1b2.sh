# C1 after the fold/prior/pack index fixes: GPU tests, bench, ncu --set full of the split fused kernel
mkdir -p gpurun_out/c1b
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/c1b/gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/c1b/gputest.log
for K in 4 8; do
timeout 300 python bench.py --config C1 --ray-split $K --no-extras --no-cpu-baseline > gpurun_out/c1b/C1_$K.json 2> gpurun_out/c1b/C1_$K.err; echo "C1 $K rc=$?"
done
timeout 300 python bench.py --config C4 --no-extras --no-cpu-baseline > gpurun_out/c1b/C4.json 2> gpurun_out/c1b/C4.err; echo "C4 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dvr_adjoint_kernel -c 1 -o gpurun_out/c1b/c1_fused python bench.py --config C1 --steps 1 --warmup 3 --graph off --no-extras --no-cpu-baseline > gpurun_out/c1b/ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/c1b/launches_C1.csv python bench.py --config C1 --steps 2 --warmup 3 --graph off --no-extras --no-cpu-baseline > gpurun_out/c1b/ncu2.log 2>&1; echo "ncu2 rc=$?"
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/c1b/*.json")):
    try:
        d = json.loads([l for l in open(f) if l.startswith("{")][-1])
        print(f.split("/")[-1], round(d["value"] / 1e9, 3), round(d["ms_per_step"], 4), d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
    except Exception as e:
        print(f, "ERR", e)
PY
