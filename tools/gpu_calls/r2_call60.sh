# C5: shapes forked on per-shape streams (default) vs serial on the caller's stream
mkdir -p gpurun_out
for r in 1 2; do
python bench.py --config c5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("fork  ", d["ms_per_step"])'
EFUNC_KIDS_SERIAL=1 python bench.py --config c5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("serial", d["ms_per_step"])'
done
