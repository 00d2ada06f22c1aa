#!/bin/bash
# Profiling pass of the current build (run under gpurun from the repo root).
#   bash scripts/profile_round.sh TAG bench   : bench (all configs) + reference arm + ncu launch lists
#   bash scripts/profile_round.sh TAG full    : one `ncu --set full` capture per top kernel
# Writes gpurun_out/prof_<tag>/...  (gpurun's ncu wrapper runs each command once without ncu first)
tag=${1:-r2}
what=${2:-bench}
out=gpurun_out/prof_$tag
mkdir -p $out
if [ "$what" = bench ]; then
  python bench.py > $out/bench.json 2> $out/bench.err
  python bench.py --impl reference > $out/bench_ref.json 2> $out/bench_ref.err
  for c in 1 2 3 4; do
    ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $out/launches_c$c.csv \
        python scripts/one_solve.py $c 1 > $out/ncu_launch_c$c.log 2>&1
  done
else
  # reports stay on the box (/tmp); the raw metric pages come back as CSV (gpurun_out/ is capped
  # at 64 MiB), plus the .ncu-rep of the kernels listed in KEEP for the source page
  KEEP=${KEEP:-"c4_hole"}
  mkdir -p /tmp/prof_$tag
  full() {  # config, kernel regex, skip, name
    ncu -f --set full --clock-control none --import-source on -k regex:"$2" -s $3 -c 1 -o /tmp/prof_$tag/full_c$1_$4 \
        python scripts/one_solve.py $1 1 > $out/ncu_full_c$1_$4.log 2>&1
    ncu -i /tmp/prof_$tag/full_c$1_$4.ncu-rep --page raw --csv > $out/full_c$1_$4.csv 2>/dev/null
    for k in $KEEP; do [ "$k" = "c$1_$4" ] && cp /tmp/prof_$tag/full_c$1_$4.ncu-rep $out/; done
  }
  full 1 "hole2d_fused_kernel" 5 hole
  full 1 "stencil2d_ym_kernel" 5 update
  full 1 "slabstep2d_kernel" 5 slabstep
  full 2 "strip_back_kernel" 5 back
  full 2 "stencil2d_ym_kernel" 5 update
  full 2 "hole2d_part_kernel" 5 lines
  full 2 "slab2d_fwd_kernel" 5 slabfwd
  full 3 "hole3d_fused_kernel" 3 hole
  full 3 "stencil3d_zm_kernel" 3 cand
  full 3 "dmma_eo2_kernel" 6 slabtransform
  full 4 "hole3d_fused_kernel" 3 hole
  full 4 "stencil3d_zm_kernel" 3 cand
  full 4 "axpy_update_kernel" 3 axpy
  full 4 "m3_apply_kernel" 3 m3apply
  full 4 "m4_kernel" 3 m4
  full 4 "skel3d_dots_rows_kernel" 3 dots
  full 4 "dmma_eo2_kernel" 6 slabtransform
  full 4 "gather_kernel" 6 gather
fi
echo done > $out/DONE_$what
