mkdir -p gpurun_out/prof_h3
for c in 4 3; do
ncu -f --set full --clock-control none --import-source on -k regex:hole3d_fused_kernel -s 3 -c 1 -o gpurun_out/prof_h3/full_c${c}_hole python scripts/one_solve.py $c 1 > gpurun_out/prof_h3/ncu_c$c.log 2>&1
ncu -i gpurun_out/prof_h3/full_c${c}_hole.ncu-rep --page raw --csv > gpurun_out/prof_h3/full_c${c}_hole.csv 2>/dev/null
done
ls -la gpurun_out/prof_h3
