# work items in two classes (heavy bricks first, light volume bricks last, Morton order within) vs one class
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_configs.py tests/test_gpu_edges_r2.py -x -q -k "fused or fit or bench or full_density or stale or r16 or tiny or large_beta or deterministic or c4 or c2" > gpurun_out/r2c48_pytest.txt 2>&1
tail -2 gpurun_out/r2c48_pytest.txt
for r in 1 2 3; do bash tools/variants.sh --no-cpu-baseline --no-e2e; done > gpurun_out/r2c48_ab.txt 2>&1
cat gpurun_out/r2c48_ab.txt
for r in 1 2; do python bench.py --config c3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("c3", d["ms_per_step"], r["frac"], r["launch_ms"])'; EFUNC_LIB_PATH=$PWD/paper_2505_21319_b200/lib/variants/cls0/libefunc.so python bench.py --config c3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("c3 cls0", d["ms_per_step"], r["frac"], r["launch_ms"])'; done
