# gather_mh with batched key loads + warp-parallel look-back scan: parity subset + A/B vs HEAD and the 3-pass scan
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or fit or det or edges or eik" > gpurun_out/r2c28_pytest.txt 2>&1
tail -2 gpurun_out/r2c28_pytest.txt
for r in 1 2; do bash tools/variants.sh --no-cpu-baseline --no-e2e; done > gpurun_out/r2c28_ab.txt 2>&1
bash tools/variants.sh --config c3 --no-cpu-baseline --no-e2e >> gpurun_out/r2c28_ab.txt 2>&1
cat gpurun_out/r2c28_ab.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r2c28_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
