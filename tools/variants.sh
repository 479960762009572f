#!/bin/bash
# Time the bench step for each library variant under lib/variants/ (tuning experiments).
# usage: bash tools/variants.sh [bench args...]
cd "$(dirname "$0")/.."
for lib in paper_2505_21319_b200/lib/libefunc.so paper_2505_21319_b200/lib/variants/*/libefunc.so; do
  r=$(EFUNC_LIB_PATH=$PWD/$lib python bench.py "$@" 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d.get("roofline",{}).get("frac"))')
  echo "$lib $r"
done
