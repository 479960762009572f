mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_configs.py tests/test_gpu_edges_r2.py -q -x --timeout 600 > gpurun_out/r2c23_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2c23_pytest.log
bash tools/variants.sh --no-cpu-baseline --no-e2e > gpurun_out/r2c23_variants.txt 2>&1
bash tools/variants.sh --no-cpu-baseline --no-e2e >> gpurun_out/r2c23_variants.txt 2>&1
tail -2 gpurun_out/r2c23_pytest.log; cat gpurun_out/r2c23_variants.txt
