#!/bin/bash
# Time the bench step for each library variant under lib/variants/ (tuning experiments).
# usage: bash tools/variants.sh [bench args...]
cd "$(dirname "$0")/.."
for lib in paper_2505_21319_b200/lib/libefunc.so paper_2505_21319_b200/lib/variants/*/libefunc.so; do
  r=$(EFUNC_LIB_PATH=$PWD/$lib python bench.py "$@" 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d.get("roofline",{}); print(round(d["ms_per_step"],4), round(r.get("frac",0),4), round(r.get("launch_ms",0),4), round(r.get("candidate_pairs_per_point",0),1))')
  echo "$lib $r"
done
