mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py -q -rA --timeout 600 > gpurun_out/r2c9_variants.log 2>&1; echo "rc=$?" >> gpurun_out/r2c9_variants.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 --deselect tests/test_gpu_variants.py > gpurun_out/r2c9_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2c9_pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2c9_bench.json 2>&1
tail -25 gpurun_out/r2c9_variants.log; tail -4 gpurun_out/r2c9_pytest_gpu.log
