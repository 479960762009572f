# k_fit occupancy with the half-warp forward (8 query-pair sums per lane): 16 warps/SM two-key backward (default),
# 16 one-key (w16b1), 20 one-key (w20b1, 96 regs), 20 two-key (w20b2), 24 one-key (w24b1, 80 regs)
mkdir -p gpurun_out
for r in 1 2; do bash tools/variants.sh --no-cpu-baseline --no-e2e; done > gpurun_out/r2c41_ab.txt 2>&1
cat gpurun_out/r2c41_ab.txt
