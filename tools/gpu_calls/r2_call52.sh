# programmatic dependent launch on the step's kernels: GPU suite, step trace, bench A/B (EFUNC_PDL=0/1)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2c52_pytest.txt 2>&1; tail -2 gpurun_out/r2c52_pytest.txt
timeout 300 python tools/step_kernels.py --steps 10 --graph > gpurun_out/r2c52_graph.txt 2>&1; grep "span" gpurun_out/r2c52_graph.txt
EFUNC_PDL=0 timeout 300 python tools/step_kernels.py --steps 10 --graph > gpurun_out/r2c52_graph_nopdl.txt 2>&1; grep "span" gpurun_out/r2c52_graph_nopdl.txt
for r in 1 2 3; do
python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("pdl  ", d["ms_per_step"], r["frac"], r["launch_ms"])'
EFUNC_PDL=0 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("nopdl", d["ms_per_step"], r["frac"], r["launch_ms"])'
done
tail -30 gpurun_out/r2c52_graph.txt
