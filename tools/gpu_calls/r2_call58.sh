# heavy class fetched from S interleaved Morton streams: S = 4 (lib), 1, 2, 8
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_configs.py -x -q -k "fused_parity_c1 or full_density or stale or pou_full" > gpurun_out/r2c58_pytest.txt 2>&1
tail -1 gpurun_out/r2c58_pytest.txt
for r in 1 2 3; do bash tools/variants.sh --no-cpu-baseline --no-e2e; done > gpurun_out/r2c58_ab.txt 2>&1
cat gpurun_out/r2c58_ab.txt
