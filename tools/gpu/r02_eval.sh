# tape-free affine walk by cell runs (bits re-evaluated per run): tests + C4 tape-free A/B
mkdir -p gpurun_out/ev
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ev/gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ev/gputest.log
V=paper_2107_12672_b200/_variants
for rep in 1 2; do
for L in product noeval; do
  if [ $L = product ]; then unset DDVR_LIB; else export DDVR_LIB=$V/libddvr_$L.so; fi
  timeout 600 python bench.py --no-band-tape --no-extras --no-cpu-baseline > gpurun_out/ev/C4nt_${L}_$rep.json 2> gpurun_out/ev/C4nt_${L}_$rep.err; echo "C4 notape $L rc=$?"
done
done
unset DDVR_LIB
timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/ev/C4tape.json 2> gpurun_out/ev/C4tape.err; echo "C4 tape rc=$?"
python - <<'PY'
import json, glob, collections
agg = collections.defaultdict(list)
for f in sorted(glob.glob("gpurun_out/ev/*.json")):
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    k = "_".join(f.split("/")[-1].split("_")[:2])
    agg[k].append((round(d["value"] / 1e9, 2), round(d["ms_per_step"], 2)))
for k, v in sorted(agg.items()):
    print(k, v)
PY
