mkdir -p gpurun_out/prof_h3
ncu -f --set full --clock-control none --import-source on -k regex:hole3d_fused_kernel -s 3 -c 1 -o gpurun_out/prof_h3/full_c4_hole python scripts/one_solve.py 4 1 > gpurun_out/prof_h3/ncu.log 2>&1
ncu -i gpurun_out/prof_h3/full_c4_hole.ncu-rep --page raw --csv > gpurun_out/prof_h3/full_c4_hole.csv 2>/dev/null
ls -la gpurun_out/prof_h3
