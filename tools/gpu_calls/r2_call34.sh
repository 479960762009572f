# k_fit CTA-chunked item fetch (FT_CHUNK = 4/8/16 items per CTA claim) vs the global per-item fetch
mkdir -p gpurun_out
EFUNC_LIB_PATH=$PWD/paper_2505_21319_b200/lib/variants/ch8/libefunc.so timeout 600 python -m pytest tests/test_gpu_bench_configs.py tests/test_gpu_parity.py -x -q -k "full_density_r32 or fused_parity_c1 or fused_matches_split_c2 or deterministic_fit_bitwise" > gpurun_out/r2c34_pytest.txt 2>&1
tail -2 gpurun_out/r2c34_pytest.txt
for r in 1 2; do bash tools/variants.sh --no-cpu-baseline --no-e2e; done > gpurun_out/r2c34_ab.txt 2>&1
cat gpurun_out/r2c34_ab.txt
