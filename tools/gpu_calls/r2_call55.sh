# ncu --set full of k_gather_queries_mh and k_query_bins (C2)
mkdir -p gpurun_out
timeout 400 ncu --set full --import-source on --clock-control none -k regex:"k_gather_queries_mh|k_query_bins|k_adamw_keys" -c 3 -f -o gpurun_out/r2s3_prep python tools/profile_step.py --steps 2 > /dev/null 2>&1
ncu -i gpurun_out/r2s3_prep.ncu-rep --page raw --csv > gpurun_out/r2s3_prep_raw.csv 2>/dev/null
ls -la gpurun_out/r2s3_prep*
