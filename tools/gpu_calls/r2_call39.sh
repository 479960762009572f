# ncu --set full of k_fit at HEAD (C2): L1/shared wavefront budget (is the L1 pipe the co-limit?)
mkdir -p gpurun_out
timeout 400 ncu --set full --import-source on --clock-control none -k regex:"k_fit$" -c 1 -f -o gpurun_out/r2s3_c2_fit python tools/profile_step.py --steps 2 > gpurun_out/r2s3_ncu.log 2>&1
tail -3 gpurun_out/r2s3_ncu.log
ncu -i gpurun_out/r2s3_c2_fit.ncu-rep --page raw --csv > gpurun_out/r2s3_c2_fit_raw.csv 2>/dev/null
ncu -i gpurun_out/r2s3_c2_fit.ncu-rep --page details --csv > gpurun_out/r2s3_c2_fit_details.csv 2>/dev/null
ls -la gpurun_out/r2s3_*
