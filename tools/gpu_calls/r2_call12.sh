mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "dense" -rA > gpurun_out/r2c12_dense.log 2>&1; echo "rc=$?" >> gpurun_out/r2c12_dense.log
timeout 900 python tools/table4.py --out gpurun_out/r2_table4.md > gpurun_out/r2c12_table4.log 2>&1
tail -5 gpurun_out/r2c12_dense.log; cat gpurun_out/r2_table4.md
