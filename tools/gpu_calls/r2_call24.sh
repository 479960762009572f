# round 2 final: bench lines of every config at HEAD, ncu captures, launch list, Table 4, inference
mkdir -p gpurun_out
timeout 400 python bench.py > gpurun_out/r2f_bench_c2.json 2> gpurun_out/r2f_bench_c2.err
for c in c1 c3 c4a c5; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2f_bench_$c.json 2> gpurun_out/r2f_bench_$c.err; done
timeout 900 python bench.py --config c4b --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_bench_c4b.json 2> gpurun_out/r2f_bench_c4b.err
timeout 400 python bench.py --deterministic --no-cpu-baseline --no-e2e > gpurun_out/r2f_bench_c2_det.json 2> gpurun_out/r2f_bench_c2_det.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2f_bench_ref.json 2> gpurun_out/r2f_bench_ref.err
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_fit$" -c 1 -f -o gpurun_out/r2f_c2_fit python tools/profile_step.py --steps 2 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_fit_eik" -c 1 -f -o gpurun_out/r2f_c3_fit_eik python tools/profile_step.py --steps 2 --J 4194304 --eikonal > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2f_launches_bench_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 python tools/table4.py --out gpurun_out/r2f_table4.md > /dev/null 2>&1
timeout 300 python tools/inference.py --fit-steps 20 > gpurun_out/r2f_inference.json 2> gpurun_out/r2f_inference.err
ls gpurun_out/r2f_*
