# group-mask A/B: parity tests of the fused path, then bench C2/C3 per variant
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or fit or det or edges" > gpurun_out/r2c26_pytest.txt 2>&1
tail -5 gpurun_out/r2c26_pytest.txt
bash tools/variants.sh --no-cpu-baseline --no-e2e > gpurun_out/r2c26_ab.txt 2>&1
bash tools/variants.sh --no-cpu-baseline --no-e2e >> gpurun_out/r2c26_ab.txt 2>&1
bash tools/variants.sh --config c4a --no-cpu-baseline --no-e2e >> gpurun_out/r2c26_ab.txt 2>&1
cat gpurun_out/r2c26_ab.txt
