# k_fit half-warp forward (FT_HALF_FWD=1: 2 keys per lane, query pairs split between the half-warps) vs FT_HALF_FWD=0
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_configs.py tests/test_gpu_edges_r2.py -x -q -k "fused or fit or bench or full_density or stale or r16 or tiny or large_beta or deterministic or c4" > gpurun_out/r2c40_pytest.txt 2>&1
tail -2 gpurun_out/r2c40_pytest.txt
for r in 1 2 3; do bash tools/variants.sh --no-cpu-baseline --no-e2e; done > gpurun_out/r2c40_ab.txt 2>&1
cat gpurun_out/r2c40_ab.txt
