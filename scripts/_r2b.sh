mkdir -p gpurun_out/prof_r2a
timeout 300 ./scripts/probe_stencil3d 509 0 > gpurun_out/probe_s3_509.txt 2>&1
timeout 300 ./scripts/probe_stencil3d 259 1 > gpurun_out/probe_s3_259.txt 2>&1
timeout 900 python bench.py > gpurun_out/prof_r2a/bench.json 2> gpurun_out/prof_r2a/bench.err
echo "bench rc=$?" >> gpurun_out/prof_r2a/bench.err
timeout 300 python bench.py --impl reference > gpurun_out/prof_r2a/bench_ref.json 2> gpurun_out/prof_r2a/bench_ref.err
for c in 1 2 3 4; do
  timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/prof_r2a/launches_c$c.csv \
      python scripts/one_solve.py $c 1 > gpurun_out/prof_r2a/ncu_launch_c$c.log 2>&1
done
bash scripts/_ab.sh ASDSM_STREAM3D=1 4 3
