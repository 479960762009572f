# fused fold + peer reduction (efunc_set_grad_peers): multirank tests, bench C2 with EFUNC_BENCH_P2P on one rank
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q > gpurun_out/r2c62_pytest.txt 2>&1; tail -3 gpurun_out/r2c62_pytest.txt
EFUNC_BENCH_NCCL1=1 EFUNC_BENCH_P2P=1 MASTER_ADDR=127.0.0.1 MASTER_PORT=29644 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2c62_bench_p2p.json 2> gpurun_out/r2c62_bench_p2p.err
python -c "import json; d=json.loads(open('gpurun_out/r2c62_bench_p2p.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['config']['launch'], d['config']['collective'], d['roofline']['frac'], d['e2e'])"
tail -3 gpurun_out/r2c62_bench_p2p.err
