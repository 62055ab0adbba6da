# sliding texel-run rows (DDVR_TF_SLIDE): GPU tests, then C1/C2 A/B against the two-row flush
mkdir -p gpurun_out/sl
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/sl/gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/sl/gputest.log
V=paper_2107_12672_b200/_variants
for rep in 1 2; do
for L in product noslide; do
  if [ $L = product ]; then unset DDVR_LIB; else export DDVR_LIB=$V/libddvr_$L.so; fi
  for C in C1 C2; do
    timeout 300 python bench.py --config $C --no-extras --no-cpu-baseline > gpurun_out/sl/${C}_${L}_$rep.json 2> gpurun_out/sl/${C}_${L}_$rep.err; echo "$C $L rc=$?"
  done
done
done
unset DDVR_LIB
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/sl/*.json")):
    try:
        d = json.loads([l for l in open(f) if l.startswith("{")][-1])
        print(f.split("/")[-1], round(d["value"] / 1e9, 3), round(d["ms_per_step"], 4), d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
    except Exception as e:
        print(f, "ERR", e)
PY
