mkdir -p gpurun_out
bash tools/variants.sh --no-cpu-baseline --no-e2e > gpurun_out/r2c8_variants.txt 2>&1
bash tools/variants.sh --no-cpu-baseline --no-e2e >> gpurun_out/r2c8_variants.txt 2>&1
python tools/kfit_mix.py > gpurun_out/r2c8_mix.txt 2>&1
EFUNC_LIB_PATH=$PWD/paper_2505_21319_b200/lib/variants/a_base/libefunc.so python tools/kfit_mix.py >> gpurun_out/r2c8_mix.txt 2>&1
cat gpurun_out/r2c8_variants.txt gpurun_out/r2c8_mix.txt
