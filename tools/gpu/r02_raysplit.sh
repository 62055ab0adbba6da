# segment-split rays (DDVR_FLAG_RAY_SPLIT_*): parity of the TF-target steps, then C1 A/B
mkdir -p gpurun_out/rs
timeout 900 python -m pytest tests/test_gpu_step_config.py -k tf_step -x -q > gpurun_out/rs/tfstep.log 2>&1; echo "tfstep rc=$?"; tail -3 gpurun_out/rs/tfstep.log
for K in 1 2 4 8 auto; do
  timeout 300 python bench.py --config C1 --ray-split $K --no-extras --no-cpu-baseline > gpurun_out/rs/C1_$K.json 2> gpurun_out/rs/C1_$K.err; echo "C1 $K rc=$?"
done
for K in 1 auto; do
  timeout 300 python bench.py --config C2 --ray-split $K --no-extras --no-cpu-baseline > gpurun_out/rs/C2_$K.json 2> gpurun_out/rs/C2_$K.err; echo "C2 $K rc=$?"
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/rs/gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/rs/gputest.log
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/rs/*.json")):
    try:
        d = json.loads([l for l in open(f) if l.startswith("{")][-1])
        print(f.split("/")[-1], round(d["value"] / 1e9, 3), round(d["ms_per_step"], 4), d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
    except Exception as e:
        print(f, "ERR", e)
PY
