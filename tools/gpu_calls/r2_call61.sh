# ncu --set full of k_fit_eik at HEAD (C3)
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_fit_eik" -c 1 -f -o gpurun_out/r2y_c3_fit_eik python tools/profile_step.py --steps 2 --J 4194304 --eikonal > /dev/null 2>&1
ncu -i gpurun_out/r2y_c3_fit_eik.ncu-rep --page raw --csv > gpurun_out/r2y_c3_fit_eik_raw.csv 2>/dev/null
ls -la gpurun_out/r2y_c3*
