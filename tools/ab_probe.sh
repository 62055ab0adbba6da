#!/bin/bash
# tools/locality_probe.py for the in-tree library and every _variants build (GPU)
for l in paper_2107_12672_b200/libddvr.so paper_2107_12672_b200/_variants/*.so; do
  echo "== $(basename $l)"; DDVR_LIB=$PWD/$l timeout 300 python tools/locality_probe.py | grep -E "^(256|320)"
done
