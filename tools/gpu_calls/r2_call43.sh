# k_fit claim-ahead (FT_CLAIM=1: next item claimed and its record copied during the backward's last rounds) vs FT_CLAIM=0
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_configs.py tests/test_gpu_edges_r2.py -x -q -k "fused or fit or bench or full_density or stale or r16 or tiny or large_beta or deterministic or c4 or tensor_core" > gpurun_out/r2c43_pytest.txt 2>&1
tail -2 gpurun_out/r2c43_pytest.txt
for r in 1 2 3; do bash tools/variants.sh --no-cpu-baseline --no-e2e; done > gpurun_out/r2c43_ab.txt 2>&1
cat gpurun_out/r2c43_ab.txt
