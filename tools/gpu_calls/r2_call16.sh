# round 2: bench lines of every config at HEAD + ncu captures of the hot kernels (profiles/r2_*)
mkdir -p gpurun_out
for c in c1 c3 c4a c5; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.err; done
timeout 900 python bench.py --config c4b --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_c4b.json 2> gpurun_out/r2_bench_c4b.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_fit$" -c 1 -f -o gpurun_out/r2_c2_fit_head python tools/profile_step.py --steps 2 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_fit_eik" -c 1 -f -o gpurun_out/r2_c3_fit_eik_head python tools/profile_step.py --steps 2 --J 4194304 --eikonal > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_dense" -c 3 -f -o gpurun_out/r2_dense_head python tools/profile_step.py --steps 1 --J 16384 --dense > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2_launches_bench_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out | tail -20
