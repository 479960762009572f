# Table 4 and inference timings at the final HEAD
mkdir -p gpurun_out
timeout 900 python tools/table4.py --out gpurun_out/r2z_table4.md > gpurun_out/r2z_table4.log 2>&1; tail -3 gpurun_out/r2z_table4.log
timeout 300 python tools/inference.py --fit-steps 20 > gpurun_out/r2z_inference.json 2> gpurun_out/r2z_inference.err; tail -c 600 gpurun_out/r2z_inference.json
cat gpurun_out/r2z_table4.md | head -20
