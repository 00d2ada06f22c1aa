timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py -x -q -p no:cacheprovider -k "3d or config3 or config4 or cfg:3 or cfg:4 or ex:4" > gpurun_out/t3d.log 2>&1
echo "tests rc=$?" >> gpurun_out/bc.txt
for pr in 0 2; do
  ASDSM_S3_PROBE=$pr timeout 300 python bench.py --config 4 --no-per-config --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/bp$pr.log 2>&1
  echo "probe $pr rc=$?" >> gpurun_out/bc.txt
done
timeout 300 python bench.py --config 3 --no-per-config --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/bc3.log 2>&1
