# FFMA2 pair math + corner-bit record order: GPU tests, then same-box A/B of the
# product build against the scalar-math variant and the previous commit's build
set -x
mkdir -p gpurun_out/f2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f2/gputest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/f2/gputest.log
V=paper_2107_12672_b200/_variants
for rep in 1 2; do
for L in new scalar head; do
  if [ $L = new ]; then unset DDVR_LIB; else export DDVR_LIB=$V/libddvr_$L.so; fi
  timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/f2/C4_${L}_$rep.json 2> gpurun_out/f2/C4_${L}_$rep.err; echo "C4 $L rc=$?"
  timeout 600 python bench.py --config C5 --views 16 --no-extras --no-cpu-baseline > gpurun_out/f2/C5_${L}_$rep.json 2> gpurun_out/f2/C5_${L}_$rep.err; echo "C5 $L rc=$?"
done
done
unset DDVR_LIB
for C in C1 C2 C3; do timeout 600 python bench.py --config $C --no-extras --no-cpu-baseline > gpurun_out/f2/${C}_new.json 2>&1; echo "$C rc=$?"; done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/f2/*.json")):
    try:
        d = json.loads([l for l in open(f) if l.startswith("{")][-1])
        print(f.split("/")[-1], round(d["value"] / 1e9, 2), d["ms_per_step"], d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
    except Exception as e:
        print(f, "ERR", e)
PY
