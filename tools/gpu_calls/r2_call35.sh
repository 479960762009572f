# k_fit strided item order (FT_SPREAD=1: items in flight spread over the domain) vs Morton order
mkdir -p gpurun_out
for r in 1 2; do bash tools/variants.sh --no-cpu-baseline --no-e2e; done > gpurun_out/r2c35_ab.txt 2>&1
cat gpurun_out/r2c35_ab.txt
