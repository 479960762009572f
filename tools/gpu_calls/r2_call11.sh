mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c11_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2c11_smoke.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -rA > gpurun_out/r2c11_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2c11_pytest_gpu.log
timeout 400 python bench.py > gpurun_out/r2c11_bench_c2.json 2> gpurun_out/r2c11_bench_c2.err
timeout 300 python tools/inference.py --fit-steps 20 > gpurun_out/r2c11_inference.json 2> gpurun_out/r2c11_inference.err
tail -3 gpurun_out/r2c11_pytest_gpu.log; tail -2 gpurun_out/r2c11_smoke.log
