# k_fit shared-memory carveout A/B: default (driver choice) vs 0 % (max L1) vs 100 % (max smem)
mkdir -p gpurun_out
for r in 1 2; do bash tools/variants.sh --no-cpu-baseline --no-e2e; done > gpurun_out/r2c33_ab.txt 2>&1
cat gpurun_out/r2c33_ab.txt
