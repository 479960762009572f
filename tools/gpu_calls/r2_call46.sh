# memset runs -> one fill kernel (k_fill_segs): GPU suite, step trace (graph), bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2c46_pytest.txt 2>&1; tail -2 gpurun_out/r2c46_pytest.txt
timeout 300 python tools/step_kernels.py --steps 10 --graph > gpurun_out/r2c46_graph.txt 2>&1; grep "span" gpurun_out/r2c46_graph.txt; tail -32 gpurun_out/r2c46_graph.txt
for r in 1 2 3; do python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["ms_per_step"], r["frac"], r["launch_ms"], d["gpu_launches"])'; done
