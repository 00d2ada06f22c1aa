mkdir -p gpurun_out/prof_src
cap() { ncu -f --set full --clock-control none --import-source on -k regex:"$2" -s $3 -c 1 -o gpurun_out/prof_src/$4 python scripts/one_solve.py $1 1 > gpurun_out/prof_src/$4.log 2>&1; }
cap 1 hole2d_fused_kernel 5 c1_hole
cap 2 hole2d_part_kernel 5 c2_lines
cap 2 strip_back_kernel 5 c2_back
cap 1 slabstep2d_kernel 5 c1_slabstep
ls -la gpurun_out/prof_src
