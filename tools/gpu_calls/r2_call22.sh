mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c22_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2c22_smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rA --durations=10 > gpurun_out/r2c22_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2c22_pytest_gpu.log
grep -E "passed|failed|FAILED" gpurun_out/r2c22_pytest_gpu.log | tail -5; tail -2 gpurun_out/r2c22_smoke.log
