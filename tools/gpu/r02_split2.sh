# tiled fold + band-march clamp trim + split variants: GPU tests, C1 split/minb A/B, C4/C5 lines
mkdir -p gpurun_out/s2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s2/gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s2/gputest.log
V=paper_2107_12672_b200/_variants
for L in product splitminb1 splitminb3 splitminb4; do
  if [ $L = product ]; then unset DDVR_LIB; else export DDVR_LIB=$V/libddvr_$L.so; fi
  for K in 4 8 16; do
    DDVR_SPLIT=$K timeout 300 python bench.py --config C1 --no-extras --no-cpu-baseline > gpurun_out/s2/C1_${L}_$K.json 2> gpurun_out/s2/C1_${L}_$K.err; echo "C1 $L $K rc=$?"
  done
done
unset DDVR_LIB
timeout 600 python bench.py --config C4 --no-extras --no-cpu-baseline > gpurun_out/s2/C4.json 2> gpurun_out/s2/C4.err; echo "C4 rc=$?"
timeout 600 python bench.py --config C5 --views 16 --no-extras --no-cpu-baseline > gpurun_out/s2/C5v16.json 2> gpurun_out/s2/C5.err; echo "C5 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/s2/launches_C1.csv python bench.py --config C1 --steps 2 --warmup 3 --graph off --no-extras --no-cpu-baseline > gpurun_out/s2/ncu2.log 2>&1; echo "ncu2 rc=$?"
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/s2/*.json")):
    try:
        d = json.loads([l for l in open(f) if l.startswith("{")][-1])
        print(f.split("/")[-1], round(d["value"] / 1e9, 3), round(d["ms_per_step"], 4), d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
    except Exception as e:
        print(f, "ERR", e)
PY
