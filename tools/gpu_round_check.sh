set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --config c3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_fit_eik" -c 1 -f -o gpurun_out/c3_fit_eik python tools/profile_step.py --steps 2 --J 4194304 --eikonal > gpurun_out/ncu_c3.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launch_c3.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
