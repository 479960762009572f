set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench tools/ubench_fp32.cu && /tmp/ubench > gpurun_out/r2_ubench.txt 2>&1
lscpu > gpurun_out/r2_lscpu.txt; nproc >> gpurun_out/r2_lscpu.txt; python -c "import os; print(len(os.sched_getaffinity(0)))" >> gpurun_out/r2_lscpu.txt
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r2_bench_c2_base.json 2> gpurun_out/r2_bench_c2_base.err
tail -2 gpurun_out/r2_ubench.txt
