# PoU full-size test with the fused-path coverage check
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "pou_full" > gpurun_out/r2c54_pytest.txt 2>&1; tail -3 gpurun_out/r2c54_pytest.txt
