# round 2, call 7: A/B of the k_fit list pipeline variants; mesh timing on a fitted-like grid
mkdir -p gpurun_out
bash tools/variants.sh --no-cpu-baseline --no-e2e > gpurun_out/r2c7_variants.txt 2>&1
bash tools/variants.sh --no-cpu-baseline --no-e2e >> gpurun_out/r2c7_variants.txt 2>&1
timeout 300 python tools/inference.py --fit-steps 20 > gpurun_out/r2c7_inference.json 2> gpurun_out/r2c7_inference.err
cat gpurun_out/r2c7_variants.txt
