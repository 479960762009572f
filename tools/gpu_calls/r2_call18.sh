mkdir -p gpurun_out
bash tools/variants.sh --no-cpu-baseline --no-e2e > gpurun_out/r2c18_variants.txt 2>&1
bash tools/variants.sh --no-cpu-baseline --no-e2e >> gpurun_out/r2c18_variants.txt 2>&1
bash tools/variants.sh --config c3 --no-cpu-baseline --no-e2e >> gpurun_out/r2c18_variants.txt 2>&1
cat gpurun_out/r2c18_variants.txt
