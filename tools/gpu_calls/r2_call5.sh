# round 2, call 5: k_fit profile at HEAD (ncu full + source), launch lists with/without k_fit_lists
mkdir -p gpurun_out
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_fit$" -c 1 -f -o gpurun_out/r2_c2_fit python tools/profile_step.py --steps 2 > gpurun_out/r2c5_ncu_fit.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_fit_lists" -c 1 -f -o gpurun_out/r2_c2_fit_lists env EFUNC_FIT_PRE=1 python tools/profile_step.py --steps 2 > gpurun_out/r2c5_ncu_lists.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2c5_launches_pre0.csv python tools/profile_step.py --steps 3 > /dev/null 2>&1
EFUNC_FIT_PRE=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2c5_launches_pre1.csv python tools/profile_step.py --steps 3 > /dev/null 2>&1
EFUNC_FIT_PRE=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2c5_bench_pre1.json 2>&1
ls -la gpurun_out
