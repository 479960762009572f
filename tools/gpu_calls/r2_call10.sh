mkdir -p gpurun_out
python tools/dbg_variant.py > gpurun_out/r2c10_dbg.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_variants.py -q -rA --timeout 600 > gpurun_out/r2c10_variants.log 2>&1; echo "rc=$?" >> gpurun_out/r2c10_variants.log
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -rA --timeout 500 > gpurun_out/r2c10_multirank.log 2>&1; echo "rc=$?" >> gpurun_out/r2c10_multirank.log
cat gpurun_out/r2c10_dbg.txt; tail -15 gpurun_out/r2c10_variants.log; tail -5 gpurun_out/r2c10_multirank.log
