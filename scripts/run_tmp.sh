mkdir -p gpurun_out/prof_eo
ncu -f --set full --clock-control none --import-source on -k regex:dmma_eo2_kernel -s 8 -c 8 -o gpurun_out/prof_eo/eo_c4 python scripts/one_solve.py 4 1 > gpurun_out/prof_eo/ncu.log 2>&1
ncu -i gpurun_out/prof_eo/eo_c4.ncu-rep --page raw --csv > gpurun_out/prof_eo/eo_c4.csv 2>/dev/null
ls -la gpurun_out/prof_eo
