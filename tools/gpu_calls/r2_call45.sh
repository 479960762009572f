# warm per-kernel timings and inter-kernel gaps of the C2 step (CUPTI via torch.profiler), eager and graph replay
mkdir -p gpurun_out
timeout 300 python tools/step_kernels.py --steps 10 > gpurun_out/r2c45_eager.txt 2>&1
timeout 300 python tools/step_kernels.py --steps 10 --graph > gpurun_out/r2c45_graph.txt 2>&1
head -3 gpurun_out/r2c45_eager.txt; cat gpurun_out/r2c45_graph.txt | head -80
