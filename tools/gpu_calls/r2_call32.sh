# k_fit at 12 warps/SM (168 registers) with/without the two-key backward unrolled 2x vs HEAD (16 warps/SM)
mkdir -p gpurun_out
for r in 1 2; do bash tools/variants.sh --no-cpu-baseline --no-e2e; done > gpurun_out/r2c32_ab.txt 2>&1
cat gpurun_out/r2c32_ab.txt
