timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py -x -q -p no:cacheprovider -k "3d or config3 or config4 or cfg:3 or cfg:4 or ex:4" > gpurun_out/t3d.log 2>&1
echo "tests rc=$?" >> gpurun_out/bc.txt
for c in 4 3; do
  timeout 300 python bench.py --config $c --no-per-config --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bc$c.log 2>&1
  echo "config $c rc=$?" >> gpurun_out/bc.txt
done
python scripts/one_solve.py 3 2 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:stream3d -s 2 -c 1 -o gpurun_out/s3prof2 python scripts/one_solve.py 3 2 > gpurun_out/ncu.log 2>&1
