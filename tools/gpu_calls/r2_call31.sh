# k_fit_tc (mma.sync 3xTF32 pair loops): parity of the fused MSE tests with EFUNC_FIT_TC=1, bench A/B
mkdir -p gpurun_out
EFUNC_FIT_TC=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_configs.py tests/test_gpu_edges_r2.py -x -q -k "fused or fit or bench or full_density or stale or r16 or tiny or large_beta or deterministic" > gpurun_out/r2c31_pytest_tc.txt 2>&1
tail -15 gpurun_out/r2c31_pytest_tc.txt
for r in 1 2; do
  python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("fp32", d["ms_per_step"], r["frac"], r["launch_ms"])'
  EFUNC_FIT_TC=1 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("tc  ", d["ms_per_step"], r["frac"], r["launch_ms"])'
done > gpurun_out/r2c31_ab.txt 2>&1
cat gpurun_out/r2c31_ab.txt
