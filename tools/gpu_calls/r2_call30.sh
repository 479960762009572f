# session 3 start: mma.sync throughput ubench, full GPU suite + bench at HEAD (restored container)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_mma tools/ubench_mma.cu && timeout 120 /tmp/ubench_mma > gpurun_out/r2c30_ubench_mma.txt 2>&1
cat gpurun_out/r2c30_ubench_mma.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2c30_pytest.txt 2>&1
tail -3 gpurun_out/r2c30_pytest.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2c30_bench.json 2> gpurun_out/r2c30_bench.err
tail -c 600 gpurun_out/r2c30_bench.json
