# register budgets of the camera/stepsize walk (POS_MINB) and the forward march (FWD_MINB): C3 A/B
mkdir -p gpurun_out/mb
V=paper_2107_12672_b200/_variants
for rep in 1 2 3; do
for L in product pos4 fwd4 fwd6; do
  if [ $L = product ]; then unset DDVR_LIB; else export DDVR_LIB=$V/libddvr_$L.so; fi
  timeout 300 python bench.py --config C3 --steps 20 --warmup 5 --no-extras --no-cpu-baseline > gpurun_out/mb/C3_${L}_$rep.json 2> gpurun_out/mb/C3_${L}_$rep.err; echo "C3 $L rc=$?"
done
done
unset DDVR_LIB
python - <<'PY'
import json, glob, collections
agg = collections.defaultdict(list)
for f in sorted(glob.glob("gpurun_out/mb/*.json")):
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    k = "_".join(f.split("/")[-1].split("_")[:2])
    agg[k].append((round(d["value"] / 1e9, 2), round(d["kernels"]["forward"]["ms"], 3), round(d["kernels"]["adjoint"]["ms"], 3)))
for k, v in sorted(agg.items()):
    print(k, v)
PY
