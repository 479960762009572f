# round 2, call 2: GPU suite (new bench-config parity, multi-rank), C2 + C3 bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -rA --durations=15 > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest_gpu.log
timeout 400 python bench.py > gpurun_out/r2_bench_c2.json 2> gpurun_out/r2_bench_c2.err
timeout 400 python bench.py --config c3 --no-cpu-baseline > gpurun_out/r2_bench_c3.json 2> gpurun_out/r2_bench_c3.err
tail -5 gpurun_out/r2_pytest_gpu.log
