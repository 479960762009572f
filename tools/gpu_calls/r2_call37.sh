# single-rank NCCL: the all-reduce captured in bench.py's step graph
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multirank.py -x -q -k nccl > gpurun_out/r2c37_pytest.txt 2>&1
tail -15 gpurun_out/r2c37_pytest.txt
EFUNC_BENCH_NCCL1=1 MASTER_ADDR=127.0.0.1 MASTER_PORT=29611 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2c37_bench_nccl1.json 2> gpurun_out/r2c37_bench_nccl1.err
tail -c 1500 gpurun_out/r2c37_bench_nccl1.json; tail -5 gpurun_out/r2c37_bench_nccl1.err
