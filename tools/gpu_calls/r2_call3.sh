# round 2, call 3: debug bench --gpus 2 (shared GPU, gloo) with a watchdog; GPU suite; C2 A/B of k_fit_lists
mkdir -p gpurun_out
EFUNC_BENCH_SHARED_GPU=1 EFUNC_BENCH_WATCHDOG=100 timeout 200 python bench.py --gpus 2 --config c1 --steps 5 --warmup 3 > gpurun_out/r2_n2dbg.out 2> gpurun_out/r2_n2dbg.err
timeout 1500 python -m pytest tests -m gpu -x -q -rA --durations=15 --deselect tests/test_gpu_multirank.py::test_bench_gpus_2_spawns_ranks_without_torchrun > gpurun_out/r2_pytest_gpu3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest_gpu3.log
EFUNC_FIT_PRE=0 timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_c2_nopre.json 2> gpurun_out/r2_bench_c2_nopre.err
timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_c2_pre.json 2> gpurun_out/r2_bench_c2_pre.err
timeout 400 python bench.py --no-cpu-baseline --no-e2e --deterministic > gpurun_out/r2_bench_c2_det.json 2> gpurun_out/r2_bench_c2_det.err
tail -5 gpurun_out/r2_pytest_gpu3.log
