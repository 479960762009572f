# work-item cost classes: K = 2 (lib) vs 1 (pure Morton), 3, 4; parity subset on K = 4
mkdir -p gpurun_out
EFUNC_LIB_PATH=$PWD/paper_2505_21319_b200/lib/variants/k4/libefunc.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_configs.py -x -q -k "fused_parity_c1 or full_density or stale or c2_full or c4a" > gpurun_out/r2c49_pytest.txt 2>&1
tail -2 gpurun_out/r2c49_pytest.txt
for r in 1 2; do bash tools/variants.sh --no-cpu-baseline --no-e2e; done > gpurun_out/r2c49_ab.txt 2>&1
cat gpurun_out/r2c49_ab.txt
