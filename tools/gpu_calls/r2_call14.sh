mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "determin" -rA > gpurun_out/r2c14_det.log 2>&1; echo "rc=$?" >> gpurun_out/r2c14_det.log
timeout 400 python bench.py --no-cpu-baseline --no-e2e --deterministic > gpurun_out/r2c14_bench_det.json 2>&1
timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2c14_bench.json 2>&1
tail -8 gpurun_out/r2c14_det.log
python -c "
import json
for f in ['gpurun_out/r2c14_bench_det.json','gpurun_out/r2c14_bench.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d['roofline']; print(f, d['ms_per_step'], r['launch_ms'], r['frac'], d['config']['path'])
"
