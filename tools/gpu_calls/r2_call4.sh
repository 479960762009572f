# round 2, call 4 (after container re-creation): GPU suite, n2 self-launch debug, C2/C3 bench, smoke
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2c4_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c4_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2c4_smoke.log
EFUNC_BENCH_SHARED_GPU=1 EFUNC_BENCH_WATCHDOG=100 timeout 200 python bench.py --gpus 2 --config c1 --steps 5 --warmup 3 > gpurun_out/r2c4_n2dbg.out 2> gpurun_out/r2c4_n2dbg.err; echo "n2 rc=$?" >> gpurun_out/r2c4_n2dbg.err
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=20 --timeout 600 --deselect tests/test_gpu_multirank.py::test_bench_gpus_2_spawns_ranks_without_torchrun > gpurun_out/r2c4_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2c4_pytest_gpu.log
timeout 400 python bench.py > gpurun_out/r2c4_bench_c2.json 2> gpurun_out/r2c4_bench_c2.err
timeout 400 python bench.py --config c3 --no-cpu-baseline > gpurun_out/r2c4_bench_c3.json 2> gpurun_out/r2c4_bench_c3.err
tail -3 gpurun_out/r2c4_pytest_gpu.log; tail -2 gpurun_out/r2c4_smoke.log; tail -2 gpurun_out/r2c4_n2dbg.err
