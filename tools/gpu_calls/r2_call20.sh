mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges_r2.py tests/test_gpu_parity.py -q -x --timeout 600 > gpurun_out/r2c20_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2c20_pytest.log
bash tools/variants.sh --no-cpu-baseline --no-e2e > gpurun_out/r2c20_variants.txt 2>&1
bash tools/variants.sh --no-cpu-baseline --no-e2e >> gpurun_out/r2c20_variants.txt 2>&1
tail -3 gpurun_out/r2c20_pytest.log; cat gpurun_out/r2c20_variants.txt
