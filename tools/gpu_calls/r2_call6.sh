# round 2, call 6: k_fit list pipeline (A/B), mesh tests, full GPU suite, inference/mesh timing
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mesh.py tests/test_gpu_bench_configs.py -q -rA > gpurun_out/r2c6_pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/r2c6_pytest_new.log
timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2c6_bench_pipe.json 2> gpurun_out/r2c6_bench_pipe.err
EFUNC_FIT_PIPE=0 timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2c6_bench_nopipe.json 2> gpurun_out/r2c6_bench_nopipe.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2c6_launches_pipe.csv python tools/profile_step.py --steps 3 > /dev/null 2>&1
timeout 300 python tools/inference.py --fit-steps 100 > gpurun_out/r2c6_inference.json 2> gpurun_out/r2c6_inference.err
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/r2c6_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2c6_pytest_gpu.log
tail -3 gpurun_out/r2c6_pytest_new.log gpurun_out/r2c6_pytest_gpu.log
