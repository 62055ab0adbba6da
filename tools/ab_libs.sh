#!/bin/bash
# A/B the experiment builds in paper_2107_12672_b200/_variants on one GPU:
#   tools/ab_libs.sh <config> [steps] [extra bench flags, e.g. --unfused]   -> gpurun_out/ab_<config>.jsonl
cfg=${1:-C4}; steps=${2:-4}; extra=${3:-}
out=gpurun_out/ab_${cfg}.jsonl; : > $out
for lib in paper_2107_12672_b200/libddvr.so paper_2107_12672_b200/_variants/*.so; do
  line=$(DDVR_LIB=$PWD/$lib timeout 600 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline $extra 2>/dev/null | tail -1)
  echo "{\"lib\": \"$(basename $lib)\", \"bench\": $line}" >> $out
done
python - "$out" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    d = json.loads(l); b = d["bench"]
    k = b.get("kernels", {})
    ks = " ".join(f"{n} {v['ms']:.2f}" for n, v in k.items() if isinstance(v, dict) and "ms" in v)
    print(f'{d["lib"]:24s} {b["value"]/1e9:8.2f} G/s  {b["ms_per_step"]:8.2f} ms  ', ks)
PY
